"""A/B timing of composite variants on one config: python tools/exp_kernels.py C 0 2 ..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
name = sys.argv[1]
kerns = [int(a) for a in sys.argv[2:]] or [0]
c = sy.CONFIGS[name]
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
out = torch.empty(r.band_shape(), dtype=torch.uint8, device="cuda")
ref = None
for kern in kerns:
    for _ in range(3):
        r.render(c.cluster_size, kernel=kern, out=out, stats=True)
    ms = []
    for _ in range(10):
        r.render(c.cluster_size, kernel=kern, out=out, stats=True)
        ms.append(r.last_stats["ms_composite"])
    img = out.clone()
    same = None if ref is None else bool(torch.equal(img, ref))
    ref = img if ref is None else ref
    ms.sort()
    print(f"kernel {kern}: composite median {ms[5]:.3f} ms min {ms[0]:.3f} total {r.last_stats['ms_total']:.2f} same_as_first={same}", flush=True)
