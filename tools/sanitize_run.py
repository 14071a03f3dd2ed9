#!/usr/bin/env python
"""Small frames for compute-sanitizer (memcheck / racecheck / synccheck):
config A at s = 1, 2, 8 (+ a band, the full-frame baseline and the paper's
thread composite) and a crop of config B's display (4K, 45 views, s = 8) with a
reduced scene, a band of tile rows.  Usage:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py [A|B|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_04509_b200 import CoherentRaster, synthetic as sy  # noqa: E402


def run_a():
    c = sy.CONFIGS["A"]
    g = CoherentRaster(0)
    g.upload_gaussians(c.make_scene())
    g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset)
    g.set_camera_rig(c.make_rig())
    for s in (1, 2, 8):
        g.render(s, stats=True)
    g.render(4, rows=(2, 6), output_format="float")
    g.render(1, fullframe=True)
    g.render(1, fullframe=True, view_batch=3)
    g.render(8, kernel=1)
    g.render(8, remap=False, kernel=1)
    g.sorted_pairs()
    g.counts(1)
    torch.cuda.synchronize()
    print("A ok", flush=True)


def run_b():
    c = sy.CONFIGS["B"]
    g = CoherentRaster(0)
    g.upload_gaussians(sy.scene_gen_v1(int(os.environ.get("CR_SAN_M", "200000")), 3, 0))
    g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset)
    g.set_camera_rig(c.make_rig())
    g.render(8, rows=(64, 70), stats=True)
    torch.cuda.synchronize()
    print("B crop ok", g.last_stats["pairs"], flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("A", "all"):
        run_a()
    if which in ("B", "all"):
        run_b()
