"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact: view map V, Psi, per-(i,k) depths and tile
counts, sorted 64-bit keys + payloads, ranges.  Images: RGB8 max |diff| <= 2
levels and float PSNR >= 50 dB (BASELINE.json north_star tolerance)."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2605_04509_b200 import synthetic as sy

pytestmark = pytest.mark.gpu


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return math.inf if mse == 0 else 10 * math.log10(1.0 / mse)


def make_pair(scene, W, H, N, Lx, slant, Koff, cams, znear=0.01, nthreads=0):
    from paper_2605_04509_b200 import CoherentRaster
    g = CoherentRaster(0)
    g.upload_gaussians(scene)
    g.set_display(W, H, N, Lx, slant, Koff)
    g.set_camera_rig(cams, znear)
    o = oracle.Oracle(nthreads=nthreads)
    o.set_scene(scene)
    o.set_display(W, H, N, Lx, slant=slant, center_offset=Koff)
    o.set_rig(cams, znear)
    return g, o


def check_frame(g, o, s, rows=None, bg=(0.0, 0.0, 0.0), kernel=None, remap=True, check_pairs=True):
    r0, r1 = rows if rows else (0, 0)
    o.render(s=s, row0=r0, row1=r1, bg=bg)
    img_f = g.render(cluster_size=s, remap=remap, kernel=kernel, background=bg,
                     output_format="float", rows=rows, stats=True).cpu().numpy()
    st = g.last_stats
    K = o.K
    assert st["num_clusters"] == K and st["bit_k"] == o.bitK
    assert st["pairs"] == o.num_pairs
    if check_pairs:
        kg, pg = g.sorted_pairs()
        ko, po = o.pairs()
        assert np.array_equal(kg, ko), "sorted keys differ"
        assert np.array_equal(pg, po), "payload order differs"
        Sg, Eg = g.ranges(K)
        So, Eo = o.ranges()
        assert np.array_equal(Sg, So) and np.array_equal(Eg, Eo)
        rec = o.records()
        vis = rec["state"] == 0
        assert np.array_equal(g.counts(K)[vis], rec["count"][vis])
        assert np.array_equal(g.counts(K)[~vis], np.zeros((~vis).sum(), np.uint32))
        assert np.array_equal(g.depths(K)[vis].view(np.uint32), rec["depth"][vis].view(np.uint32))
    ref = o.image()
    assert img_f.shape == ref.shape
    assert np.all(np.isfinite(img_f))
    p = psnr(np.clip(img_f, 0, 1), np.clip(ref, 0, 1))
    assert p >= 50.0, f"PSNR {p:.2f} dB"
    img8 = g.render(cluster_size=s, remap=remap, kernel=kernel, background=bg,
                    output_format="rgb8", rows=rows).cpu().numpy()
    ref8 = oracle.quantize_rgb8(ref)
    d = np.abs(img8.astype(np.int16) - ref8.astype(np.int16))
    assert d.max() <= 2, f"max RGB8 diff {d.max()}"
    return img_f, p


@pytest.fixture(scope="module")
def cfgA_pair():
    _need_gpu()
    c = sy.CONFIGS["A"]
    return make_pair(c.make_scene(), c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset,
                     c.make_rig())


def test_view_map_and_remap_bit_exact(cfgA_pair):
    g, o = cfgA_pair
    assert np.array_equal(g.view_map(), o.view_map())
    assert np.array_equal(g.remap_table(), o.remap(1))


@pytest.mark.parametrize("W,H,N,Lx,slant,K", [
    (3840, 2160, 100, 19.6153, math.atan(0.1852), 7.3),
    (3840, 2160, 45, 19.6153, math.atan(0.1852), 7.3),
    (250, 138, 71, 12.37, -0.2, -5.5),
    (1, 1, 3, 3.0, 0.0, 0.0),
])
def test_view_map_remap_displays(W, H, N, Lx, slant, K):
    _need_gpu()
    from paper_2605_04509_b200 import CoherentRaster
    g = CoherentRaster(0)
    g.set_display(W, H, N, Lx, slant, K)
    o = oracle.Oracle()
    o.set_display(W, H, N, Lx, slant=slant, center_offset=K)
    assert np.array_equal(g.view_map(), o.view_map())
    assert np.array_equal(g.remap_table(), o.remap(1))


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_config_a_parity(cfgA_pair, s):
    g, o = cfgA_pair
    check_frame(g, o, s, bg=(0.05, 0.1, 0.2))


def test_config_a_kernels_and_remap_agree(cfgA_pair):
    # Psi only permutes independent writes: staged (remap) == thread
    # (remap) == thread (raster order), bit for bit.
    g, o = cfgA_pair
    a = g.render(8, remap=True, kernel=0, output_format="float").cpu().numpy()
    b = g.render(8, remap=True, kernel=1, output_format="float").cpu().numpy()
    c = g.render(8, remap=False, kernel=1, output_format="float").cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(b, c)


def test_band_shards_equal_full_frame(cfgA_pair):
    g, o = cfgA_pair
    full = g.render(4, output_format="float").cpu().numpy()
    kf, pf = g.sorted_pairs()
    bands = [(0, 3), (3, 4), (4, 9)]
    parts = []
    for r0, r1 in bands:
        parts.append(g.render(4, output_format="float", rows=(r0, r1)).cpu().numpy())
        kb, pb = g.sorted_pairs()
        t = (kb >> np.uint64(32 + 1)) // np.uint64(16)
        sel = ((kf >> np.uint64(33)) // np.uint64(16) >= r0) & ((kf >> np.uint64(33)) // np.uint64(16) < r1)
        assert np.array_equal(kb, kf[sel]) and np.array_equal(pb, pf[sel])
        assert np.all((t >= r0) & (t < r1))
    assert np.array_equal(np.concatenate(parts), full)
    # and the band frames match the oracle
    check_frame(g, o, 4, rows=(3, 7))


def test_ragged_panel_and_deg3():
    _need_gpu()
    W, H, N = 250, 138, 13  # clipped edge tiles in x and y
    sc = sy.random_scene(3000, 3, seed=9, scale_median=0.04)
    cams = sy.orbit_rig(N, 10.0, W, H, radius=3.0, height=0.4, fov_y_deg=50.0)
    g, o = make_pair(sc, W, H, N, 11.3, 0.17, 3.3, cams)
    for s in (1, 5):
        check_frame(g, o, s, bg=(0.3, 0.3, 0.3))
    check_frame(g, o, 5, rows=(2, 9))


def test_identical_pose_rig_any_s_equals_s1():
    _need_gpu()
    W, H, N = 128, 80, 8
    sc = sy.random_scene(2000, 1, seed=3, scale_median=0.05)
    cams = sy.identical_rig(N, W, H, radius=3.0, height=0.3, fov_y_deg=50.0)
    g, o = make_pair(sc, W, H, N, 9.7, 0.2, 1.0, cams)
    ref = g.render(1, output_format="float", stats=True).cpu().numpy()
    P1 = g.last_stats["pairs"]
    for s in (2, 4, 8):
        img = g.render(s, output_format="float", stats=True).cpu().numpy()
        assert np.array_equal(img, ref)
        assert g.last_stats["pairs"] * N == P1 * (N // s)


def test_empty_scene_and_near_plane():
    _need_gpu()
    W, H, N = 64, 48, 4
    cams = sy.orbit_rig(N, 5.0, W, H, radius=2.0, height=0.0)
    g, o = make_pair(sy.empty_scene(0), W, H, N, 7.0, 0.1, 0.0, cams)
    img = g.render(2, background=(0.25, 0.5, 1.0), output_format="float").cpu().numpy()
    assert np.all(img == np.array([0.25, 0.5, 1.0], np.float32))
    # Gaussians straddling / behind the camera and huge ones: culling paths
    sc = sy.random_scene(500, 0, seed=4, extent=2.5, scale_median=0.3)
    g.upload_gaussians(sc)
    o.set_scene(sc)
    check_frame(g, o, 2)


def test_device_upload_equals_host_upload(cfgA_pair):
    g, o = cfgA_pair
    c = sy.CONFIGS["A"]
    sc = c.make_scene()
    a = g.render(8, output_format="float").cpu().numpy()
    g.upload_gaussians({k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v)
                        for k, v in sc.items()})
    b = g.render(8, output_format="float").cpu().numpy()
    assert np.array_equal(a, b)


def test_host_output_buffer(cfgA_pair):
    g, o = cfgA_pair
    dev = g.render(8).cpu().numpy()
    host = np.zeros_like(dev)
    g.render(8, out=host)
    assert np.array_equal(dev, host)


def test_error_codes():
    _need_gpu()
    from paper_2605_04509_b200 import CoherentRaster
    from paper_2605_04509_b200._native import CrError
    g = CoherentRaster(0)
    with pytest.raises(CrError, match="NOT_READY"):
        g.render(8)
    with pytest.raises(CrError, match="INVALID_CONFIG"):
        g.set_display(100, 100, 0, 5.0, 0.1, 0.0)
    with pytest.raises(CrError, match="INVALID_CONFIG"):
        g.set_display(100, 100, 300, 5.0, 0.1, 0.0)
    g.set_display(64, 48, 4, 5.0, 0.1, 0.0)
    with pytest.raises(CrError, match="CONFIG_MISMATCH"):
        g.set_camera_rig(sy.orbit_rig(3, 5.0, 64, 48))
    g.set_camera_rig(sy.orbit_rig(4, 5.0, 64, 48))
    bad = sy.random_scene(10, 0, 0)
    bad["means"][3, 1] = np.nan
    with pytest.raises(CrError, match="NONFINITE"):
        g.upload_gaussians(bad)
    g.upload_gaussians(sy.random_scene(10, 0, 0))
    with pytest.raises(CrError, match="INVALID_CONFIG"):
        g.render(33)
    with pytest.raises(CrError, match="INVALID_ARG"):
        g.render(2, rows=(2, 1))


def test_config_b_full_size_sampled_tiles():
    # BASELINE configs[1] at full size (1M Gaussians SH3, 45 views, 4K): bit-exact
    # pair count and per-(i,k) counts for the whole frame, exact keys and images on
    # a sample of tiles the oracle composites one by one.
    _need_gpu()
    c = sy.CONFIGS["B"]
    g, o = make_pair(c.make_scene(), c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset,
                     c.make_rig())
    rng = np.random.default_rng(0)
    TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
    tiles = np.sort(rng.choice(TX * TY, 48, replace=False)).astype(np.int32)
    o.render(s=8, tiles=tiles)
    img = g.render(8, output_format="float", stats=True).cpu().numpy()
    st = g.last_stats
    assert st["pairs"] == int(o.records()["count"].sum())
    kg, pg = g.sorted_pairs()
    tg = (kg >> np.uint64(32 + o.bitK)).astype(np.int64)
    sel = np.isin(tg, tiles)
    ko, po = o.pairs()
    assert np.array_equal(kg[sel], ko) and np.array_equal(pg[sel], po)
    ref = o.image()
    for t in tiles:
        tx, ty = t % TX, t // TX
        a = img[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        b = ref[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        assert np.abs(a - b).max() <= 2.0 / 255
    a = np.concatenate([img[(t // TX) * 16:(t // TX + 1) * 16, (t % TX) * 16:(t % TX + 1) * 16]
                        for t in tiles])
    b = np.concatenate([ref[(t // TX) * 16:(t // TX + 1) * 16, (t % TX) * 16:(t % TX + 1) * 16]
                        for t in tiles])
    assert psnr(np.clip(a, 0, 1), np.clip(b, 0, 1)) >= 50.0


def _sampled_tile_check(g, o, cfg, s, tiles, rows=None):
    TX = (cfg.W + 15) // 16
    r0, r1 = rows if rows else (0, 0)
    o.render(s=s, row0=r0, row1=r1, tiles=tiles)
    img = g.render(s, output_format="float", stats=True, rows=rows).cpu().numpy()
    st = g.last_stats
    assert st["pairs"] == int(o.records()["count"].sum())
    kg, pg = g.sorted_pairs()
    tg = (kg >> np.uint64(32 + o.bitK)).astype(np.int64)
    sel = np.isin(tg, tiles)
    ko, po = o.pairs()
    assert np.array_equal(kg[sel], ko) and np.array_equal(pg[sel], po)
    ref = o.image()
    y0 = r0 * 16
    a = np.concatenate([img[(t // TX) * 16 - y0:(t // TX + 1) * 16 - y0, (t % TX) * 16:(t % TX + 1) * 16]
                        for t in tiles])
    b = np.concatenate([ref[(t // TX) * 16 - y0:(t // TX + 1) * 16 - y0, (t % TX) * 16:(t % TX + 1) * 16]
                        for t in tiles])
    assert np.abs(a - b).max() <= 2.0 / 255
    assert psnr(np.clip(a, 0, 1), np.clip(b, 0, 1)) >= 50.0
    # the RGB8 output the bench times, on the same tiles
    img8 = g.render(s, rows=rows).cpu().numpy()
    a8 = np.concatenate([img8[(t // TX) * 16 - y0:(t // TX + 1) * 16 - y0, (t % TX) * 16:(t % TX + 1) * 16]
                         for t in tiles]).astype(np.int16)
    assert np.abs(a8 - oracle.quantize_rgb8(b).astype(np.int16)).max() <= 2
    return st


def test_config_c_full_size_sampled_tiles():
    # the bench workload itself (BASELINE configs[2]: 3M Gaussians SH3, 100 views,
    # 4K, s=8) in the launch configuration bench.py times: exact pair count, exact
    # keys/payloads and images on sampled tiles (denser middle rows included)
    _need_gpu()
    c = sy.CONFIGS["C"]
    g, o = make_pair(c.make_scene(), c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset,
                     c.make_rig())
    TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
    rng = np.random.default_rng(1)
    rows = rng.choice(np.arange(40, 100), 8, replace=False)
    tiles = np.sort(np.concatenate([rows * TX + rng.integers(0, TX, 8),
                                    rng.choice(TX * TY, 16, replace=False)])).astype(np.int32)
    tiles = np.unique(tiles)
    st = _sampled_tile_check(g, o, c, 8, tiles)
    assert st["pairs"] > 1e8
    # a balanced band of the 8-rank split, same checks
    band = (68, 74)
    tb = np.unique(np.array([ty * TX + tx for ty in range(*band) for tx in (0, 37, 120, 239)],
                            np.int32))
    _sampled_tile_check(g, o, c, 8, tb, rows=band)


def test_config_e_head_tracked_pose_sampled_tiles():
    # BASELINE configs[4] at its benchmarked size: a head-tracked pose of the
    # 45-view 4K display with the full 3M-Gaussian scene
    _need_gpu()
    c = sy.CONFIGS["E"]
    pose = sy.head_tracked_poses(256, seed=1)[7]
    scene = c.make_scene()
    g, o = make_pair(scene, c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset,
                     c.make_rig(**pose))
    TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
    tiles = np.unique(np.random.default_rng(2).choice(TX * TY, 24, replace=False)).astype(np.int32)
    _sampled_tile_check(g, o, c, 8, tiles)


def test_config_d_8k_sampled_tiles():
    # BASELINE configs[3] at its benchmarked size (6M Gaussians, 7680x4320, 100
    # views: 17 tile-id bits, 3 tile radix passes), one frame, sampled tiles
    _need_gpu()
    c = sy.CONFIGS["D"]
    scene = c.make_scene()
    g, o = make_pair(scene, c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.make_rig())
    TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
    rng = np.random.default_rng(3)
    tiles = np.unique(np.concatenate([rng.choice(TX * TY, 16, replace=False),
                                      (TY // 2) * TX + rng.integers(0, TX, 8)])).astype(np.int32)
    _sampled_tile_check(g, o, c, 8, tiles)


def test_determinism_repeated_frames(cfgA_pair):
    g, o = cfgA_pair
    a = g.render(4, output_format="float").cpu().numpy()
    ka, pa = g.sorted_pairs()
    for _ in range(3):
        b = g.render(4, output_format="float").cpu().numpy()
        kb, pb = g.sorted_pairs()
        assert np.array_equal(a, b) and np.array_equal(ka, kb) and np.array_equal(pa, pb)


def test_fullframe_baseline_equals_subpixel_s1(cfgA_pair):
    # N1: rendering every view full frame and interlacing by V gives,
    # subpixel by subpixel, the s=1 subpixel render (same lists, same blend ops),
    # and matches the oracle's brute force (full frame per view + interlace).
    g, o = cfgA_pair
    sub = g.render(1, output_format="float").cpu().numpy()
    ff = g.render(1, output_format="float", fullframe=True, stats=True).cpu().numpy()
    assert np.array_equal(sub, ff)
    o.render(s=1)
    bf = o.bruteforce()
    assert np.abs(ff - bf).max() <= 2.0 / 255 and psnr(np.clip(ff, 0, 1), np.clip(bf, 0, 1)) >= 50
    band = g.render(1, output_format="rgb8", fullframe=True, rows=(2, 6)).cpu().numpy()
    assert np.array_equal(band, g.render(1, output_format="rgb8", rows=(2, 6)).cpu().numpy())
    # s > 1: every view full frame with its cluster's attributes, interlaced ==
    # the subpixel path at the same s (same lists, means and blend arithmetic)
    assert np.array_equal(g.render(4, output_format="float", fullframe=True).cpu().numpy(),
                          g.render(4, output_format="float").cpu().numpy())


def test_fullframe_view_batches(cfgA_pair):
    # the paper's batched full-frame 3DGS baseline ("3DGS (batch=B)", P:520;
    # B=1 plain 3DGS): views rendered B per pass (own preprocess, binning and
    # sort per pass) then interlaced once == all views in one pass, bit for bit
    g, o = cfgA_pair
    for s in (1, 2):
        ref = g.render(s, output_format="float", fullframe=True).cpu().numpy()
        ref_v = g.render(s, output_format="rgb8", view_frames=True, rows=(1, 5)).cpu().numpy()
        for vb in (1, 3, 4, 6):
            if vb % s:
                continue
            got = g.render(s, output_format="float", fullframe=True, view_batch=vb, stats=True)
            assert np.array_equal(got.cpu().numpy(), ref)
            got_v = g.render(s, output_format="rgb8", view_frames=True, rows=(1, 5), view_batch=vb)
            assert np.array_equal(got_v.cpu().numpy(), ref_v)
    host = np.zeros(g.band_shape(None), np.uint8)
    g.render(1, output_format="rgb8", fullframe=True, view_batch=3, out=host)
    assert np.array_equal(host, g.render(1, output_format="rgb8", fullframe=True).cpu().numpy())
    from paper_2605_04509_b200._native import CrError
    with pytest.raises(CrError):
        g.render(2, fullframe=True, view_batch=3)  # not a multiple of the cluster size


@pytest.mark.parametrize("s", [16, 18, 3])
def test_large_and_odd_clusters(s):
    """Cluster sizes beyond 8: G = 16 (P2K's s=16) and G = 32 (P4K's s=18)
    lane groups, and a non-power-of-two s=3 (G=4 with an idle lane), against
    the oracle: bit-exact keys/ranges/counts, image tolerance; plus a band."""
    _need_gpu()
    W, H, N = 192, 112, 40
    sc = sy.random_scene(3000, 1, seed=21, scale_median=0.035)
    cams = sy.orbit_rig(N, 20.0, W, H, radius=3.0, height=0.3, fov_y_deg=50.0)
    g, o = make_pair(sc, W, H, N, 13.7, 0.19, 2.1, cams)
    check_frame(g, o, s)
    check_frame(g, o, s, rows=(2, 5))


def test_big_footprints_general_path():
    """Records beyond the 64-byte union slot (> 6 union rows or >= 64 tile
    columns) take the warp-wide general path (k_count_big / k_emit_big):
    large splats on a wide panel, bit-exact against the oracle."""
    _need_gpu()
    W, H, N = 1280, 112, 12
    sc = sy.random_scene(600, 0, seed=5, scale_median=0.25)
    cams = sy.orbit_rig(N, 12.0, W, H, radius=3.0, height=0.2, fov_y_deg=30.0)
    g, o = make_pair(sc, W, H, N, 10.9, 0.21, 0.7, cams)
    for s in (4, 12):
        check_frame(g, o, s)
        g.render(cluster_size=s, stats=True)
        assert g.last_stats["emit_fallback"] > 0, "general path not exercised"
    check_frame(g, o, 4, rows=(1, 5))


def test_parallel_camera_rig_motion_bound():
    """A camera-array rig (pure translation between views, no rotation): every
    cluster's rotation bound is 0, so the pre-cull takes the rigid-motion-bound
    path (one projection per record); the result must still be bit-exact,
    full frame and in a band."""
    _need_gpu()
    W, H, N = 256, 144, 16
    sc = sy.random_scene(4000, 1, seed=17, scale_median=0.03)
    cams = sy.identical_rig(N, W, H, radius=3.0, height=0.3, fov_y_deg=50.0).copy()
    cams[:, 9] += np.linspace(-0.12, 0.12, N, dtype=np.float32)  # camera-space x offsets
    g, o = make_pair(sc, W, H, N, 11.3, 0.19, 1.7, cams)
    for s in (4, 8):
        check_frame(g, o, s)
    check_frame(g, o, 8, rows=(3, 6))


def test_wide_depth_range_uncompressed_presort():
    """Depths spanning 0.05 .. 1e9 with K = 16 clusters: the compressed
    (k, depth - min) presort key needs more than 32 bits, so the presort falls
    back to a 32-bit depth sort plus a stable cluster pass; still bit-exact."""
    _need_gpu()
    W, H, N = 192, 112, 16
    rng = np.random.default_rng(23)
    n = 3000
    sc = sy.random_scene(n, 0, seed=23, scale_median=0.03)
    cams = sy.orbit_rig(N, 12.0, W, H, radius=3.0, height=0.0, fov_y_deg=50.0)
    # spread the Gaussians along the rig's viewing direction, log-uniform in depth
    zc = np.exp(rng.uniform(np.log(0.05), np.log(1e9), n))
    dirs = sc["means"] / np.maximum(np.linalg.norm(sc["means"], axis=1, keepdims=True), 1e-6)
    eye = np.array([0.0, 0.0, 3.0])
    means = eye[None, :] + (np.array([0.0, 0.0, -1.0])[None, :] + 0.3 * dirs) * zc[:, None]
    sc["means"] = means.astype(np.float32)
    sc["scales"] = (sc["scales"] * np.maximum(zc, 1.0)[:, None] * 0.3).astype(np.float32)
    g, o = make_pair(sc, W, H, N, 9.9, 0.21, 0.4, cams)
    check_frame(g, o, 1)
    check_frame(g, o, 2)


@pytest.mark.parametrize("name", ["P2K", "P4K"])
def test_paper_display_panels_sampled_tiles(name):
    # the paper's own display setups at full size — 63 views on the
    # 1440x2560 portrait panel at s=16 and 71 views on 3840x2160 at s=18 (P:392,
    # P:473-474) with the 3M-Gaussian scene; exact keys, images on sampled tiles
    _need_gpu()
    c = sy.CONFIGS[name]
    g, o = make_pair(c.make_scene(), c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset,
                     c.make_rig())
    TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
    rng = np.random.default_rng(11)
    tiles = np.unique(np.concatenate([rng.choice(TX * TY, 16, replace=False),
                                      (TY // 2) * TX + rng.integers(0, TX, 8)])).astype(np.int32)
    _sampled_tile_check(g, o, c, c.cluster_size, tiles)


def test_async_host_output(cfgA_pair):
    # CR_FLAG_ASYNC_OUT: frames copied to pinned host buffers on the copy
    # stream (double-buffered device staging) equal the synchronous renders
    g, o = cfgA_pair
    c = sy.CONFIGS["A"]
    rigs = [c.make_rig(), sy.orbit_rig(c.N, 6.0, c.W, c.H, radius=3.2, height=0.1, fov_y_deg=50.0),
            c.make_rig()]
    ref = []
    for cams in rigs:
        g.set_camera_rig(cams)
        ref.append(g.render(4, output_format="rgb8").cpu().numpy())
    hosts = [torch.empty(g.band_shape(None), dtype=torch.uint8, pin_memory=True) for _ in rigs]
    for cams, h in zip(rigs, hosts):
        g.set_camera_rig(cams)
        g.render(4, output_format="rgb8", out=h.numpy(), async_out=True)
    g.synchronize()
    for h, r_ in zip(hosts, ref):
        assert np.array_equal(h.numpy(), r_)
    g.set_camera_rig(c.make_rig())


@pytest.mark.parametrize("name,s,rows", [("A", 8, None), ("A", 1, None), ("A", 3, (2, 5)),
                                         ("B", 8, (60, 64)), ("P4K", 18, (40, 43))])
def test_pairs_composite_equals_one_subpixel_per_lane(monkeypatch, name, s, rows):
    # k_composite_pairs (two subpixels of one view per lane, packed fp32x2 blend,
    # view runs padded to even length) against k_composite_staged (CR_EXP bit 6):
    # same per-subpixel operations in the same order, so frames (float and RGB8)
    # and evaluation counts must be identical; rows exercise the tile split path
    _need_gpu()
    from paper_2605_04509_b200 import CoherentRaster
    c = sy.CONFIGS[name]
    scene = c.make_scene()
    out = {}
    for exp in ("0", "64"):
        monkeypatch.setenv("CR_EXP", exp)
        g = CoherentRaster(0)
        g.upload_gaussians(scene)
        g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset)
        g.set_camera_rig(c.make_rig())
        f = g.render(s, output_format="float", rows=rows, background=(0.1, 0.2, 0.3)).cpu().numpy()
        b = g.render(s, output_format="rgb8", rows=rows).cpu().numpy()
        g.render(s, rows=rows, stats=True, count_evals=True)
        out[exp] = (f, b, g.last_stats["evals"])
        g.close()
    assert np.array_equal(out["0"][0], out["64"][0])
    assert np.array_equal(out["0"][1], out["64"][1])
    assert out["0"][2] == out["64"][2]
