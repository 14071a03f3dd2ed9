"""A/B timing harness: python tools/exp_variants.py C 0 [1 2 ...]

Renders the config with each value of the CR_EXP environment variable (an
experiment knob a kernel-variant A/B build can read in cr_render_interlaced;
the committed library ignores it), prints median per-stage ms and whether the
image equals the first variant's (variants must be bit-identical)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
name = sys.argv[1]
exps = [int(a) for a in sys.argv[2:]] or [0]
c = sy.CONFIGS[name]
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
out = torch.empty(r.band_shape(), dtype=torch.uint8, device="cuda")
ref = None
for rep in range(2):
    for ex in exps:
        os.environ["CR_EXP"] = str(ex)
        for _ in range(3):
            r.render(c.cluster_size, out=out, stats=True)
        st = []
        for _ in range(10):
            r.render(c.cluster_size, out=out, stats=True)
            st.append(dict(r.last_stats))
        img = out.clone()
        same = None
        if ref is None:
            ref = img
        else:
            same = bool(torch.equal(img, ref))
        med = lambda k: sorted(s[k] for s in st)[len(st) // 2]
        print(f"exp {ex:3d}: total {med('ms_total'):7.3f}  pre {med('ms_preprocess'):6.3f}  bin {med('ms_bin'):6.3f}"
              f"  sort {med('ms_sort'):6.3f}  comp {med('ms_composite'):6.3f}  same_image={same}", flush=True)
