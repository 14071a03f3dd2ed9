"""GPU: the row-bucketed binning tail (cr_rowbin.cuh — row entries, stable
sort by tile row, per-row stable sort by tile column) produces exactly the
lists of the emission + 2-pass LSD tile sort (Eq.11 key order; Alg.2
GenerateKeys P:791-808), and both match the oracle.  The LSD tail is forced
with CR_EXP bit 3 (read when a context is created); panels wider than 512
tile columns take it by default.  CR_EXP bit 4 starts the big-record entry
store at 64 entries so the grow-and-redo path runs."""
import os

import numpy as np
import pytest
import torch

from paper_2605_04509_b200 import CoherentRaster
from paper_2605_04509_b200 import synthetic as sy
from test_gpu_parity import _need_gpu, check_frame, make_pair

pytestmark = pytest.mark.gpu


def _ctx(exp, scene, W, H, N, Lx, slant, Koff, cams):
    old = os.environ.get("CR_EXP")
    os.environ["CR_EXP"] = str(exp)
    try:
        g = CoherentRaster(0)
    finally:
        if old is None:
            del os.environ["CR_EXP"]
        else:
            os.environ["CR_EXP"] = old
    g.upload_gaussians(scene)
    g.set_display(W, H, N, Lx, slant, Koff)
    g.set_camera_rig(cams)
    return g


def _frame(g, s, rows=None):
    img = g.render(cluster_size=s, output_format="float", rows=rows, stats=True).cpu().numpy()
    K = g.last_stats["num_clusters"]
    k, p = g.sorted_pairs()
    S, E = g.ranges(K)
    return img, k, p, S, E, g.counts(K), dict(g.last_stats)


def _same(a, b):
    for x, y in zip(a[:6], b[:6]):
        assert np.array_equal(x, y)
    assert a[6]["pairs"] == b[6]["pairs"]


@pytest.mark.parametrize("name,s", [("A", 8), ("A", 1), ("A", 3)])
def test_rowbin_equals_lsd_tail(name, s):
    _need_gpu()
    c = sy.CONFIGS[name]
    args = (c.make_scene(), c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.make_rig())
    _same(_frame(_ctx(0, *args), s), _frame(_ctx(8, *args), s))


def test_rowbin_big_records_store_regrow():
    # big records (> 6 union rows or >= 64 columns) put their row entries in
    # the big store; starting it at 64 entries forces the grow-and-redo path
    _need_gpu()
    W, H, N = 1280, 112, 12
    sc = sy.random_scene(600, 0, seed=5, scale_median=0.25)
    cams = sy.orbit_rig(N, 12.0, W, H, radius=3.0, height=0.2, fov_y_deg=30.0)
    args = (sc, W, H, N, 10.9, 0.21, 0.7, cams)
    ref = _frame(_ctx(8, *args), 4)
    assert ref[6]["emit_fallback"] > 8
    _same(_frame(_ctx(16, *args), 4), ref)
    _same(_frame(_ctx(0, *args), 4), ref)
    _same(_frame(_ctx(0, *args), 4, rows=(1, 5)), _frame(_ctx(8, *args), 4, rows=(1, 5)))


def test_wide_panel_takes_lsd_tail_and_matches_oracle():
    # 8320 px = 520 tile columns > 512: the emission + LSD tail, vs the oracle
    _need_gpu()
    W, H, N = 8320, 48, 6
    sc = sy.random_scene(3000, 0, seed=47, scale_median=0.02)
    cams = sy.orbit_rig(N, 6.0, W, H, radius=3.0, height=0.2, fov_y_deg=20.0)
    g, o = make_pair(sc, W, H, N, 13.1, 0.17, 1.3, cams)
    check_frame(g, o, 3)
