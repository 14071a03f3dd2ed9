"""GPU edge cases (round 2): configurations just outside round 1's tested
envelope, each against the CPU oracle through the C ABI — the maximum view
count N = 255 at s = 1 and 2 (K up to 255 clusters, up to K + 24 composite
work items per tile), a panel taller than 16 * 288 px with a splat whose
cluster tile union spans more than 288 tile rows (windowed big-record
emission), N = 1, the degenerate-covariance cull count, and the upload error
path keeping the previous scene (header: "on error the context keeps its
previous state")."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_04509_b200 import synthetic as sy
from test_gpu_parity import _need_gpu, check_frame, make_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 24, 32])
def test_max_views_255(s):
    # P:246 N views; the ABI's maximum N = 255 (u8 view map).  At s=1 every
    # view is its own cluster (K = 255, Bit_K = 8): a 16x16 tile holds up to
    # K + 24 cluster-aligned chunks, far beyond round 1's 128-chunk cap.  Every
    # count lane/view split runs with 255 cameras (20 KB) in dynamic shared
    # memory on top of its static arrays (past the default 48 KB per block).
    _need_gpu()
    W, H, N = 256, 144, 255
    sc = sy.random_scene(1500, 1, seed=41, scale_median=0.04)
    cams = sy.orbit_rig(N, 40.0, W, H, radius=3.0, height=0.2, fov_y_deg=50.0)
    g, o = make_pair(sc, W, H, N, 41.3, 0.13, 3.7, cams)
    check_frame(g, o, s, bg=(0.1, 0.0, 0.2))


def test_tall_panel_union_over_288_rows():
    # 256 x 4864 px (TY = 304 > 288 rows of k_emit_big's per-warp arrays): one
    # large splat close to the cameras covers the full height, so its cluster
    # union has > 288 tile rows and is emitted window by window.
    _need_gpu()
    W, H, N = 256, 4864, 4
    sc = sy.random_scene(60, 0, seed=43, scale_median=0.02)
    sc["means"][0] = [0.0, 0.0, 0.6]
    sc["scales"][0] = [0.05, 2.0, 0.05]
    sc["quats"][0] = [1, 0, 0, 0]
    sc["opacities"][0] = 0.9
    cams = sy.orbit_rig(N, 4.0, W, H, radius=3.0, height=0.0, fov_y_deg=60.0)
    g, o = make_pair(sc, W, H, N, 7.7, 0.11, 0.9, cams)
    o.render(s=2, composite=False)
    rec = o.records()
    assert rec["count"].max() > 2 * 288  # some union spans > 288 rows (x >= 2 columns)
    check_frame(g, o, 2)
    g.render(2, stats=True)
    assert g.last_stats["emit_fallback"] > 0


def test_single_view_display():
    # N = 1 (degenerate display: V == 0 everywhere, K = 1, Bit_K = 1): plain 3DGS
    _need_gpu()
    W, H = 120, 72
    sc = sy.random_scene(800, 1, seed=45, scale_median=0.05)
    cams = sy.orbit_rig(1, 0.0, W, H, radius=3.0, height=0.3, fov_y_deg=50.0)
    g, o = make_pair(sc, W, H, 1, 6.1, 0.2, 0.0, cams)
    check_frame(g, o, 1)
    check_frame(g, o, 8)  # s > N: one padded cluster, representative view 0


def test_degenerate_cull_count_matches_oracle():
    # O6 / S:342: a covariance that overflows fp32 is culled as degenerate in
    # every cluster, counted in cr_stats.culled_degenerate like the oracle's state 3.
    _need_gpu()
    W, H, N = 96, 64, 4
    sc = sy.random_scene(300, 0, seed=47, scale_median=0.05)
    sc["scales"][:5] = 3e19
    cams = sy.orbit_rig(N, 6.0, W, H, radius=3.0, height=0.2)
    g, o = make_pair(sc, W, H, N, 5.5, 0.1, 0.0, cams)
    check_frame(g, o, 2)
    g.render(2, stats=True)
    o.render(s=2, composite=False)
    assert g.last_stats["culled_degenerate"] == int((o.records()["state"] == 3).sum()) >= 10


def test_rejected_upload_keeps_previous_scene(cfgA_pair_local):
    from paper_2605_04509_b200._native import CrError
    g, c = cfgA_pair_local
    ref = g.render(8, output_format="float").cpu().numpy()
    bad = c.make_scene()
    bad["sh"][17, 0, 1] = np.inf
    with pytest.raises(CrError, match="NONFINITE"):
        g.upload_gaussians(bad)
    bad2 = c.make_scene()
    bad2["opacities"][3] = 1.5
    with pytest.raises(CrError, match="INVALID_ARG"):
        g.upload_gaussians(bad2)
    again = g.render(8, output_format="float").cpu().numpy()
    assert np.array_equal(ref, again)


@pytest.fixture(scope="module")
def cfgA_pair_local():
    _need_gpu()
    from paper_2605_04509_b200 import CoherentRaster
    c = sy.CONFIGS["A"]
    g = CoherentRaster(0)
    g.upload_gaussians(c.make_scene())
    g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset)
    g.set_camera_rig(c.make_rig())
    return g, c


def test_wide_panel_8320px():
    # 8320 px wide (520 tile columns over 3 tile rows: the tile sort's high
    # digit spans few values and its histogram is aggregated), vs the oracle
    _need_gpu()
    W, H, N = 8320, 48, 6
    sc = sy.random_scene(3000, 0, seed=47, scale_median=0.02)
    cams = sy.orbit_rig(N, 6.0, W, H, radius=3.0, height=0.2, fov_y_deg=20.0)
    g, o = make_pair(sc, W, H, N, 13.1, 0.17, 1.3, cams)
    check_frame(g, o, 3)


@pytest.mark.parametrize("W,H", [(256, 144), (250, 138)])
def test_tile_split_equals_whole_tile_composite(W, H):
    # small grids split each tile's chunks over several CTAs that store their
    # subpixels directly; CR_EXP bit 5 forces one CTA per tile (shared-memory
    # tile + 16-byte row stores, scalar at the ragged edge): identical frames
    _need_gpu()
    import os
    from paper_2605_04509_b200 import CoherentRaster
    sc = sy.random_scene(4000, 1, seed=49, scale_median=0.04)
    cams = sy.orbit_rig(8, 8.0, W, H, radius=3.0, height=0.2, fov_y_deg=50.0)
    imgs = []
    for exp in ("0", "32"):
        old = os.environ.get("CR_EXP")
        os.environ["CR_EXP"] = exp
        try:
            g = CoherentRaster(0)
        finally:
            if old is None:
                del os.environ["CR_EXP"]
            else:
                os.environ["CR_EXP"] = old
        g.upload_gaussians(sc)
        g.set_display(W, H, 8, 12.5, 0.25, 1.5)
        g.set_camera_rig(cams)
        for fmt in ("float", "rgb8"):
            imgs.append(g.render(cluster_size=4, output_format=fmt).cpu().numpy())
            imgs.append(g.render(cluster_size=4, output_format=fmt, rows=(2, 6)).cpu().numpy())
    for a, b in zip(imgs[:4], imgs[4:]):
        assert np.array_equal(a, b)


def test_orbit_rig_bands_equal_full_frame():
    # config C's display and orbit rig (narrow clusters: the per-axis
    # rigid-motion bound pre-cull, and in bands the lazy-SH pre-test before
    # the exact EWA) with a reduced scene_gen v1 scene: every band's sorted
    # pairs are the full frame's filtered to its rows and the band images
    # tile the full frame bit for bit
    _need_gpu()
    from paper_2605_04509_b200 import CoherentRaster
    c = sy.CONFIGS["C"]
    g = CoherentRaster(0)
    g.upload_gaussians(sy.scene_gen_v1(200_000, 3, seed=3))
    g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
    g.set_camera_rig(c.make_rig())
    full = g.render(8, output_format="rgb8").cpu().numpy()
    kf, pf = g.sorted_pairs()
    tf = (kf >> np.uint64(32 + 4)) // np.uint64(240)  # Bit_K = 4 (K = 13), TX = 240
    for r0, r1 in [(0, 9), (40, 47), (66, 71), (120, 135)]:
        band = g.render(8, output_format="rgb8", rows=(r0, r1)).cpu().numpy()
        assert np.array_equal(band, full[r0 * 16:r1 * 16])
        kb, pb = g.sorted_pairs()
        sel = (tf >= r0) & (tf < r1)
        assert np.array_equal(kb, kf[sel]) and np.array_equal(pb, pf[sel])


def test_17bit_tile_ids_nine_bit_first_pass():
    # 8192 x 2064 px = 512 x 129 tiles: 17-bit tile ids, sorted in 2 passes
    # with a 9-bit first digit; bit-identical to 3 passes of 8-bit digits
    # (CR_EXP bit 3), and a band of it against the oracle
    _need_gpu()
    import os
    from paper_2605_04509_b200 import CoherentRaster
    W, H, N = 8192, 2064, 6
    sc = sy.random_scene(20000, 1, seed=53, scale_median=0.03)
    cams = sy.orbit_rig(N, 6.0, W, H, radius=3.0, height=0.2, fov_y_deg=40.0)
    res = []
    for exp in ("0", "8"):
        old = os.environ.get("CR_EXP")
        os.environ["CR_EXP"] = exp
        try:
            g = CoherentRaster(0)
        finally:
            if old is None:
                del os.environ["CR_EXP"]
            else:
                os.environ["CR_EXP"] = old
        g.upload_gaussians(sc)
        g.set_display(W, H, N, 13.3, 0.17, 2.1)
        g.set_camera_rig(cams)
        img = g.render(3, output_format="rgb8", stats=True).cpu().numpy()
        k, p = g.sorted_pairs()
        res.append((img, k, p, g.last_stats["pairs"]))
    assert res[0][3] == res[1][3] > 100000
    for a, b in zip(res[0][:3], res[1][:3]):
        assert np.array_equal(a, b)
    g, o = make_pair(sc, W, H, N, 13.3, 0.17, 2.1, cams)
    check_frame(g, o, 3, rows=(60, 64))
