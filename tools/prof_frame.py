"""Render a few frames of a config for profiling (ncu): python tools/prof_frame.py C [frames] [s] [kernel]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
name = sys.argv[1] if len(sys.argv) > 1 else "C"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = int(sys.argv[3]) if len(sys.argv) > 3 else 8
kern = int(sys.argv[4]) if len(sys.argv) > 4 else 0
remap = bool(int(sys.argv[5])) if len(sys.argv) > 5 else True
rows = tuple(int(v) for v in sys.argv[6].split(":")) if len(sys.argv) > 6 else None
c = sy.CONFIGS[name]
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
out = torch.empty(r.band_shape(rows), dtype=torch.uint8, device="cuda")
for f in range(frames):
    r.render(s, kernel=kern, remap=remap, out=out, stats=True, rows=rows)
    print(f, r.last_stats, flush=True)
torch.cuda.synchronize()
