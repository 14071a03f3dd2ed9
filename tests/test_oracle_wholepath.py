"""Whole-path pins for the oracle (round 2): quantities that only cro_render
computes — camera centre / SH view direction / colour clamp, the conic
inversion, the Eq.11 key packing, the degenerate cull — checked against
closed forms and independent constructions, plus the superfluous-keys
invariant and a dense-sampling check that the shipped O7
form never under-estimates a tile set.  CPU only.

Each test was run against planted mutations of oracle/oracle.cpp (C = -R t,
reversed view direction, colour clamp removed, conic B sign flipped, A<->C
swapped, k shifted in the key, degenerate cull removed): every mutation fails
at least one test here (profiles/r02/oracle_mutations.txt).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from paper_2605_04509_b200 import synthetic as sy

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
SH_C0 = 0.28209479177387814  # S:77 / S:80 (3DGS real SH, l = 0)
SH_C1 = 0.4886025119029199   # S:81 (l = 1)


def _one_gaussian(mu, quat, scales, opacity, sh):
    sh = np.asarray(sh, np.float32)
    deg = int(round(math.sqrt(sh.shape[0]))) - 1
    return dict(means=np.asarray([mu], np.float32), quats=np.asarray([quat], np.float32),
                scales=np.asarray([scales], np.float32),
                opacities=np.asarray([opacity], np.float32), sh=sh[None].copy(), sh_degree=deg)


def _sigma2d_independent(cam, mu, quat, scales):
    """Sigma2D = J W Sigma W^T J^T + 0.3 I in fp64 (Eq.10 input):
    Sigma from scipy's rotation of the quaternion, J by central differences of the
    pinhole map — nothing here reuses the oracle's formulas."""
    R = cam[:9].reshape(3, 3).astype(np.float64)
    t = cam[9:12].astype(np.float64)
    fx, fy, cx, cy = [float(v) for v in cam[12:]]
    Rq = Rotation.from_quat(np.asarray(quat, np.float64)[[1, 2, 3, 0]]).as_matrix()
    Sig = Rq @ np.diag(np.asarray(scales, np.float64) ** 2) @ Rq.T
    p = R @ np.asarray(mu, np.float64) + t

    def pi(pp):
        return np.array([fx * pp[0] / pp[2] + cx, fy * pp[1] / pp[2] + cy])

    J = np.zeros((2, 3))
    for a in range(3):
        e = np.zeros(3)
        e[a] = 1e-6 * max(1.0, abs(p[a]))
        J[:, a] = (pi(p + e) - pi(p - e)) / (2 * e[a])
    return J @ R @ Sig @ R.T @ J.T + 0.3 * np.eye(2), pi(p)


def _closed_form_image(W, H, m2d, S2, o, col, bg):
    """One Gaussian, front-to-back (Eqs.9-10): C = c a + bg (1 - a) where
    a = min(0.99, o exp(-d^T S2^-1 d / 2)) >= 1/255, else C = bg."""
    Si = np.linalg.inv(S2)
    ys, xs = np.mgrid[0:H, 0:W]
    dx = xs + 0.5 - m2d[0]
    dy = ys + 0.5 - m2d[1]
    q = Si[0, 0] * dx * dx + 2 * Si[0, 1] * dx * dy + Si[1, 1] * dy * dy
    a = np.minimum(0.99, o * np.exp(-0.5 * q))
    img = np.empty((H, W, 3))
    for u in range(3):
        img[..., u] = np.where(a >= 1 / 255, col[u] * a + bg[u] * (1 - a), bg[u])
    near_thr = np.abs(a - 1 / 255) < 2e-5 * (1 / 255) * 50  # alpha at the 1/255 test: either side
    return img, near_thr


@pytest.mark.parametrize("rig", ["single", "identical8"])
def test_single_anisotropic_gaussian_whole_path_closed_form(rig):
    # North star: "a single Gaussian matches its closed-form footprint" — rendered
    # through cro_render (tiles, keys, sort, ranges, composite) at N=1, s=1 and on
    # an identical-pose rig N=8, s=8 (every view sees the same footprint).
    W, H = 96, 64
    mu = [0.05, -0.03, 0.1]
    quat = [0.95, 0.05, 0.1, 0.3]  # rotated: b != 0, a != c in Sigma2D
    scales = [0.2, 0.06, 0.02]
    o_ = 0.85
    dc = np.array([0.8, -0.5, 1.2])
    sh = dc[None, :]
    cam = sy.look_at_camera([0.3, 0.2, 3.0], [0, 0, 0], [0, 1, 0], 80.0, 80.0, 48.0, 32.0)
    N, s = (1, 1) if rig == "single" else (8, 8)
    orc = oracle.Oracle(nthreads=2)
    orc.set_scene(_one_gaussian(mu, quat, scales, o_, sh))
    orc.set_display(W, H, N, 7.3, slant=0.2, center_offset=1.1)
    orc.set_rig(np.repeat(cam[None], N, axis=0))
    bg = (0.1, 0.2, 0.3)
    orc.render(s=s, bg=bg)
    img = orc.image().astype(np.float64)
    S2, m2d = _sigma2d_independent(cam, mu, quat, scales)
    assert abs(S2[0, 1]) > 0.05 * math.sqrt(S2[0, 0] * S2[1, 1])  # really anisotropic + rotated
    assert abs(S2[0, 0] - S2[1, 1]) > 0.05 * S2[0, 0]
    col = np.maximum(SH_C0 * dc + 0.5, 0.0)
    ref, amb = _closed_form_image(W, H, m2d, S2, o_, col, bg)
    d = np.abs(img - ref)
    d[amb] = 0.0
    assert d.max() <= 2e-4, f"max |oracle - closed form| = {d.max():.3g}"
    covered = np.any(np.abs(ref - np.asarray(bg)) > 1e-3, axis=2).sum()
    assert covered > 150  # the footprint spans several tiles
    assert orc.num_pairs >= 4 * (N // s)


def test_sh_colour_view_direction_and_clamp_through_render():
    # O11 (Pi_SH of Eq.6): colour = max(SH(dir) + 0.5, 0) with dir the unit
    # vector from the representative camera's CENTRE to the mean.  The centres are the
    # known eye positions of two look-at cameras (not derived from R, t here), and the
    # only non-zero coefficient is the x band (index 3, basis -C1 x).
    mu = np.array([0.2, 0.1, -0.3])
    h3 = np.array([1.0, -2.0, 0.3])  # channel 1 goes negative from eye_a: the clamp
    sh = np.zeros((4, 3))
    sh[3] = h3
    eyes = [np.array([3.0, 0.4, 0.5]), np.array([-2.5, -0.3, 1.8])]
    W, H = 64, 48
    cams = np.stack([sy.look_at_camera(e, [0, 0, 0], [0, 1, 0], 60.0, 60.0, 32.0, 24.0)
                     for e in eyes])
    orc = oracle.Oracle(nthreads=1)
    orc.set_scene(_one_gaussian(mu, [1, 0, 0, 0], [0.02] * 3, 0.9, sh))
    orc.set_display(W, H, 2, 5.0, slant=0.0, center_offset=0.0)
    orc.set_rig(cams)
    orc.render(s=1)
    rec = orc.records()
    assert np.all(rec["state"][:, 0] == 0)
    clamped = 0
    for k, e in enumerate(eyes):
        d = (mu - e) / np.linalg.norm(mu - e)
        raw = 0.5 - SH_C1 * d[0] * h3
        exp = np.maximum(raw, 0.0)
        clamped += int(np.sum(raw < 0))
        assert np.allclose(rec["color"][k, 0], exp, atol=2e-6), (k, rec["color"][k, 0], exp)
    assert clamped >= 1  # the clamp branch is exercised


def test_conic_is_inverse_of_sigma2d():
    # Eq.10: the conic is Sigma2D^-1 = [[A, B], [B, C]] — checked with a
    # numpy inverse of the records' own (a, b, c) on rotated anisotropic Gaussians.
    o, _ = _setup_random(seed=31)
    o.render(s=2, composite=False)
    rec = o.records()
    vis = rec["state"] == 0
    cv = rec["cov2d"][vis].astype(np.float64)
    cn = rec["conic"][vis].astype(np.float64)
    assert cv.shape[0] > 500
    n_aniso = 0
    for (a, b, c, det), (A, B, C) in zip(cv, cn):
        inv = np.linalg.inv(np.array([[a, b], [b, c]]))
        sc = np.max(np.abs(inv))
        assert abs(A - inv[0, 0]) <= 1e-5 * sc and abs(C - inv[1, 1]) <= 1e-5 * sc
        assert abs(B - inv[0, 1]) <= 1e-5 * sc
        n_aniso += abs(b) > 0.05 * math.sqrt(a * c) and abs(a - c) > 0.05 * a
    assert n_aniso > 100


def _setup_random(M=600, W=96, H=64, N=8, seed=0, scale=0.06):
    sc = sy.random_scene(M, 1, seed, scale_median=scale)
    o = oracle.Oracle(nthreads=4)
    o.set_scene(sc)
    o.set_display(W, H, N, 9.3, slant=0.21, center_offset=2.2)
    o.set_rig(sy.orbit_rig(N, 8.0, W, H, radius=3.0, height=0.3, fov_y_deg=50.0))
    return o, sc


def test_spec_key_example_through_render():
    # S:365 (Eq.11): K=8 clusters, Bit_K=3, tile 5, cluster 2, depth 1.0f
    # -> key 181453979648.  Eight identical cameras (R = I, t = 0) put one small
    # Gaussian at camera depth exactly 1.0 inside tile 5 of a 128x32 panel, so
    # cro_render emits one pair per cluster k with key t<<35 | k<<32 | bits(1.0f).
    ex = GOLD["keys"][0]
    N, W, H = 8, 128, 32
    cam = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 100.0, 100.0, 88.0, 8.0], np.float32)
    orc = oracle.Oracle(nthreads=1)
    orc.set_scene(_one_gaussian([0.0, 0.0, 1.0], [1, 0, 0, 0], [0.001] * 3, 0.9,
                                np.zeros((1, 3))))
    orc.set_display(W, H, N, 5.0, slant=0.0, center_offset=0.0)
    orc.set_rig(np.repeat(cam[None], N, axis=0))
    orc.render(s=1, composite=False)
    assert orc.K == ex["K"] and orc.bitK == ex["bitK"]
    keys, pay = orc.pairs()
    assert keys.size == N and np.all(pay == 0)
    assert int(keys[ex["k"]]) == ex["expect"]
    assert keys.tolist() == [(5 << 35) | (k << 32) | 0x3F800000 for k in range(N)]


def test_superfluous_keys_do_not_change_the_image():
    # P:379-382 / S:392: the cluster tile union holds pairs a given view never
    # uses; growing every tile rectangle of the tile test by 2 px adds more such
    # pairs (alpha < 1/255 at every pixel centre of the tile) and changes the
    # image by at most 1e-2 (in practice only at the exp-vs-tau boundary).
    o, _ = _setup_random(M=500, seed=33)
    o.render(s=4, bg=(0.2, 0.1, 0.05))
    P0, img0 = o.num_pairs, o.image()
    o.set_tile_pad(2.0)
    o.render(s=4, bg=(0.2, 0.1, 0.05))
    P2, img2 = o.num_pairs, o.image()
    o.set_tile_pad(0.0)
    assert P2 > P0 * 1.05
    d = np.abs(img2 - img0)
    assert d.max() <= 1e-2
    assert np.count_nonzero(d) <= 3


def test_accutile_shipped_form_never_underestimates_dense_sampling():
    # O7 as shipped (xr/xl via one rounded reciprocal 1/c, DESIGN.md §3 Z11/O7):
    # points sampled densely inside the ellipse {d^T Sigma^-1 d <= tau(1 - 1e-5)}
    # that fall on a tile's pixel-centre rectangle must find that tile listed, over
    # 1500 random ellipses (anisotropic, rotated, sub-pixel to ~60 px, off-screen
    # parts) — the "never under-estimates" property re-checked for this form.
    rng = np.random.default_rng(8)
    TX, TY = 14, 10
    hits = 0
    for _ in range(1500):
        m = rng.uniform(-30, 16 * TX + 30, 2).astype(np.float32)
        sa, sb = np.exp(rng.uniform(-1.5, 4.2, 2))
        th = rng.uniform(0, np.pi)
        Rm = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        Sig = Rm @ np.diag([sa ** 2, sb ** 2]) @ Rm.T + 0.3 * np.eye(2)
        a, b, c = np.float32(Sig[0, 0]), np.float32(Sig[0, 1]), np.float32(Sig[1, 1])
        det = np.float32(np.float32(a * c) - np.float32(b * b))
        if not det > 0:
            continue
        tau = np.float32(rng.uniform(0.2, 11.0))
        tiles = set(oracle.tileset(m, (a, b, c, det), tau, TX, TY).tolist())
        S = np.array([[a, b], [b, c]], np.float64)
        L = np.linalg.cholesky(S)
        # uniform samples in the unit disc, mapped into the ellipse, plus its boundary
        n = 4000
        r = np.sqrt(rng.random(n))
        ph = rng.uniform(0, 2 * np.pi, n)
        disc = np.stack([r * np.cos(ph), r * np.sin(ph)], 1)
        ring = np.stack([np.cos(np.linspace(0, 2 * np.pi, 720)), np.sin(np.linspace(0, 2 * np.pi, 720))], 1)
        u = np.concatenate([disc, ring]) * math.sqrt(float(tau) * (1 - 1e-5))
        pts = m.astype(np.float64) + u @ L.T
        fx = pts[:, 0] - 0.5
        fy = pts[:, 1] - 0.5
        tx = np.floor(fx / 16).astype(np.int64)
        ty = np.floor(fy / 16).astype(np.int64)
        on_rect = (fx - 16 * tx <= 15.0) & (fy - 16 * ty <= 15.0)
        ok = on_rect & (tx >= 0) & (tx < TX) & (ty >= 0) & (ty < TY)
        need = set((ty[ok] * TX + tx[ok]).tolist())
        missing = need - tiles
        assert not missing, (m, (a, b, c, det), tau, sorted(missing)[:5])
        hits += len(need)
    assert hits > 3000


def test_degenerate_covariance_is_culled_and_counted():
    # O6 / S:342: det(Sigma2D) <= 0 (or undefined) culls (i,k) as degenerate.  A
    # Gaussian whose covariance overflows fp32 (scale 3e19 -> s^2 = 9e38 > FLT_MAX)
    # has no finite footprint: culled in every cluster, no pairs, background image.
    # A thin but regular needle next to it stays (det = 0.3 tr + 0.09 > 0).
    sc = sy.random_scene(2, 0, 0)
    sc["means"][:] = [[0.0, 0.0, 0.0], [0.05, 0.0, 0.0]]
    sc["quats"][:] = [[1, 0, 0, 0], [0.9, 0.1, 0.3, 0.2]]
    sc["scales"][:] = [[3e19, 3e19, 3e19], [0.2, 1e-4, 1e-4]]
    sc["opacities"][:] = [0.9, 0.9]
    orc = oracle.Oracle(nthreads=1)
    orc.set_scene(sc)
    orc.set_display(64, 48, 4, 5.0, slant=0.1, center_offset=0.0)
    orc.set_rig(sy.orbit_rig(4, 6.0, 64, 48, radius=3.0, height=0.2))
    orc.render(s=2, bg=(0.3, 0.3, 0.3))
    st = orc.records()["state"]
    assert np.all(st[:, 0] == 3)  # degenerate in both clusters
    assert np.all(st[:, 1] == 0)
    keys, pay = orc.pairs()
    assert keys.size > 0 and np.all(pay == 1)
