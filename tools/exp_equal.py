"""Two CR_EXP developer switches render bit-identical frames (float and RGB8)
and sorted (key, payload) pairs:
python tools/exp_equal.py C 0 4 [s]"""
import os, subprocess, sys
cfg, ea, eb = sys.argv[1], sys.argv[2], sys.argv[3]
s = sys.argv[4] if len(sys.argv) > 4 else ""
code = r'''
import os, sys, hashlib
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
c = sy.CONFIGS[sys.argv[1]]
s = int(sys.argv[2]) if sys.argv[2] else c.cluster_size
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
h = hashlib.sha1()
for fmt in ("float", "rgb8"):
    h.update(r.render(s, output_format=fmt).cpu().numpy().tobytes())
r.render(s, stats=True, count_evals=True)
k, p = r.sorted_pairs()
h.update(k.tobytes()); h.update(p.tobytes())
print(h.hexdigest(), r.last_stats["evals"], r.last_stats["pairs"])
'''
outs = []
for e in (ea, eb):
    res = subprocess.run([sys.executable, "-c", code, cfg, s], env=dict(os.environ, CR_EXP=e),
                         capture_output=True, text=True, timeout=600)
    outs.append(res.stdout.strip())
    print(f"CR_EXP={e}: {outs[-1]} {res.stderr[-300:]}")
print("EQUAL" if outs[0] == outs[1] and outs[0] else "DIFFERENT")
