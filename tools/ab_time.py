"""Per-stage frame timing of one config (median of N frames, CUDA events via
cr_stats): python tools/ab_time.py C [frames] [s]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_04509_b200 import CoherentRaster, synthetic as sy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
c = sy.CONFIGS[name]
s = int(sys.argv[3]) if len(sys.argv) > 3 else c.cluster_size
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
out = torch.empty(r.band_shape(), dtype=torch.uint8, device="cuda")
for _ in range(3):
    r.render(s, out=out)
st = []
for _ in range(n):
    r.render(s, out=out, stats=True)
    st.append(dict(r.last_stats))
med = lambda k: sorted(x[k] for x in st)[len(st) // 2]  # noqa: E731
print(f"{name} s={s}: total {med('ms_total'):.3f} ms  pre {med('ms_preprocess'):.3f}  "
      f"bin {med('ms_bin'):.3f}  sort {med('ms_sort'):.3f}  comp {med('ms_composite'):.3f}  "
      f"pairs {st[-1]['pairs']}  launches {st[-1]['launches']}", flush=True)
