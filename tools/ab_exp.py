"""A/B of CR_EXP developer switches (read at context creation): per-stage
median frame times for each value.  python tools/ab_exp.py C 0,1,2 [rows r0:r1]"""
import os
import subprocess
import sys

cfg = sys.argv[1]
exps = sys.argv[2].split(",")
rows = sys.argv[3] if len(sys.argv) > 3 else ""
code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
c = sy.CONFIGS[sys.argv[1]]
rows = tuple(int(v) for v in sys.argv[2].split(":")) if len(sys.argv) > 2 and sys.argv[2] else None
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
for _ in range(3): r.render(c.cluster_size, rows=rows)
st = []
for _ in range(15):
    r.render(c.cluster_size, rows=rows, stats=True); st.append(dict(r.last_stats))
med = lambda k: sorted(x[k] for x in st)[len(st) // 2]
print(f"exp={os.environ.get('CR_EXP')} {sys.argv[1]} rows={rows}: total {med('ms_total'):.3f} pre {med('ms_preprocess'):.3f} bin {med('ms_bin'):.3f} sort {med('ms_sort'):.3f} comp {med('ms_composite'):.3f}", flush=True)
'''
for rep in range(2):
    for e in exps:
        env = dict(os.environ, CR_EXP=e)
        subprocess.run([sys.executable, "-c", code, cfg, rows], env=env)
