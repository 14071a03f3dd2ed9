"""Row-bucketed tail vs emission + LSD tail (CR_EXP bit 3) on one config:
identical sorted pairs, ranges and image.  python tools/rb_check.py A [s]"""
import os, subprocess, sys
cfg = sys.argv[1] if len(sys.argv) > 1 else "A"
code = r'''
import os, sys, hashlib
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
c = sy.CONFIGS[sys.argv[1]]
s = int(sys.argv[2]) if len(sys.argv) > 2 else c.cluster_size
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
img = r.render(s, output_format="float", stats=True).cpu().numpy()
st = dict(r.last_stats)
k, p = r.sorted_pairs()
S, E = r.ranges(st["num_clusters"])
h = hashlib.sha1()
for a in (k, p, S, E, img): h.update(np.ascontiguousarray(a).tobytes())
print(os.environ.get("CR_EXP", "0"), h.hexdigest(), st["pairs"], st["ms_bin"], st["ms_sort"], st["ms_total"], flush=True)
'''
for e in ("8", "0"):
    env = dict(os.environ, CR_EXP=e)
    subprocess.run([sys.executable, "-c", code] + sys.argv[1:], env=env, timeout=600)
