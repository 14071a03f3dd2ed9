"""Where the row-bucketed tail and the LSD tail differ (debug): python tools/rb_diff.py A [s]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy


def ctx(exp, c):
    os.environ["CR_EXP"] = str(exp)
    g = CoherentRaster(0)
    g.upload_gaussians(c.make_scene())
    g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
    g.set_camera_rig(c.make_rig())
    return g


c = sy.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "A"]
s = int(sys.argv[2]) if len(sys.argv) > 2 else c.cluster_size
out = {}
for e in (8, 0):
    g = ctx(e, c)
    res = []
    for f in range(3):
        img = g.render(s, output_format="float", stats=True).cpu().numpy()
        st = dict(g.last_stats)
        print(e, f, {k: round(v, 3) if isinstance(v, float) else v for k, v in st.items() if k.startswith("ms") or k in ("pairs", "emit_fallback")}, flush=True)
    K = st["num_clusters"]
    k, p = g.sorted_pairs()
    S, E = g.ranges(K)
    out[e] = dict(img=img, k=k, p=p, S=S, E=E, cnt=g.counts(K))
for name in ("k", "p", "S", "E", "cnt", "img"):
    a, b = out[8][name], out[0][name]
    if a.shape != b.shape:
        print(name, "shape", a.shape, b.shape)
        continue
    d = np.nonzero((a != b).reshape(-1))[0]
    print(name, "ndiff", len(d), "first", d[:8], a.reshape(-1)[d[:8]], b.reshape(-1)[d[:8]], flush=True)
