"""Debug: per-(i,k) tile counts of the GPU vs the oracle on config E pose 7
(the sampled-tile test's frame); prints mismatching records."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
c = sy.CONFIGS["E"]
pose = sy.head_tracked_poses(256, seed=1)[7]
scene = c.make_scene()
cams = c.make_rig(**pose)
g = CoherentRaster(0)
g.upload_gaussians(scene)
g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset)
g.set_camera_rig(cams, 0.01)
o = oracle.Oracle()
o.set_scene(scene)
o.set_display(c.W, c.H, c.N, c.lens_pitch, slant=c.slant, center_offset=c.center_offset)
o.set_rig(cams, 0.01)
TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
tiles = np.unique(np.random.default_rng(2).choice(TX * TY, 24, replace=False)).astype(np.int32)
o.render(s=8, tiles=tiles, composite=False)
g.render(cluster_size=8, stats=True)
K = o.K
gc = g.counts(K)
rec = o.records()
oc = rec["count"]
vis = rec["state"] == 0
print("lib", os.environ.get("CR_LIB"), "pairs gpu", g.last_stats["pairs"], "oracle", int(oc.sum()))
bad = np.nonzero((gc != oc) & vis)
print("mismatching records", len(bad[0]))
for k, i in list(zip(*bad))[:10]:
    print(" k", k, "i", i, "gpu", gc[k, i], "oracle", oc[k, i], "mean", scene["means"][i], "scale", scene["scales"][i])
