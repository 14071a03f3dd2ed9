"""Pins for the oracle's geometry: O3 clusters, O4 upload constants, O5 mean
projection (Eq.5), O6 EWA covariance (Eq.6 Pi_cov), O7 AccuTile tile sets and
O9 key layout (Eq.11).  CPU only."""
import json
import math
import os
import struct

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from paper_2605_04509_b200 import synthetic as sy

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ O3
@pytest.mark.parametrize("ex", GOLD["clusters"])
def test_clusters_spec_examples(ex):
    K, bitK, rep = oracle.clusters(ex["N"], ex["s"])
    assert K == ex["K"], ex["cite"]
    if "rep0" in ex:
        assert rep[0] == ex["rep0"]
    if "reps" in ex:
        assert rep == ex["reps"]


def test_clusters_padding_and_bitk():
    # N=100, s=8 -> K=13, last cluster padded: rep(12) = min(96+4, 99) = 99 (Z6)
    K, bitK, rep = oracle.clusters(100, 8)
    assert (K, bitK) == (13, 4) and rep[12] == 99 and rep[0] == 4
    assert oracle.clusters(8, 8)[1] == 1  # Bit_K = max(1, ceil(log2 1))
    assert oracle.clusters(16, 2)[1] == 3
    assert oracle.clusters(17, 2)[1] == 4
    for N in range(1, 40):
        for s in range(1, 12):
            K, b, rep = oracle.clusters(N, s)
            assert K == -(-N // s) and (1 << b) >= K and b >= 1
            assert all(k * s <= rep[k] < N for k in range(K))


# ------------------------------------------------------------------ O4
@pytest.mark.parametrize("ex", GOLD["covariance"])
def test_covariance_spec_examples(ex):
    cov, _ = oracle.gaussian_constants(np.array([ex["quat_wxyz"]]), np.array([ex["scale"]]),
                                       np.array([0.5]))
    m = cov[0]
    full = np.array([[m[0], m[1], m[2]], [m[1], m[3], m[4]], [m[2], m[4], m[5]]])
    assert np.allclose(full, np.diag(ex["expect_diag"]), atol=1e-6), ex["cite"]


def test_covariance_vs_scipy_rotation_and_sign_flip():
    rng = np.random.default_rng(1)
    q = rng.standard_normal((500, 4)) * rng.uniform(0.2, 3, (500, 1))  # unnormalised
    s = np.exp(rng.normal(-3, 1, (500, 3)))
    cov, tau = oracle.gaussian_constants(q, s, rng.uniform(0.01, 1, 500))
    cov2, _ = oracle.gaussian_constants(-q, s, np.full(500, 0.5))
    assert np.array_equal(cov, cov2)  # q -> -q invariance
    R = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()  # scipy wants (x,y,z,w)
    ref = R @ (np.eye(3)[None] * (s ** 2)[:, None, :]) @ np.transpose(R, (0, 2, 1))
    got = np.stack([cov[:, [0, 1, 2]], cov[:, [1, 3, 4]], cov[:, [2, 4, 5]]], 1)
    scale = np.max(s ** 2, axis=1)[:, None, None]
    assert np.all(np.abs(got - ref) <= 1e-6 * scale)


def test_tau_is_alpha_threshold():
    o = np.array([1.0, 0.5, 1 / 255.0, 0.001], np.float32)
    _, tau = oracle.gaussian_constants(np.tile([1, 0, 0, 0], (4, 1)), np.ones((4, 3)), o)
    # o*exp(-tau/2) = 1/255  <=>  tau = 2 ln(255 o); tau <= 0 when o <= 1/255
    assert np.allclose(o[:2] * np.exp(-tau[:2] / 2), 1 / 255.0, rtol=1e-6)
    assert tau[2] <= 1e-6 and tau[3] < 0


# ------------------------------------------------------------------ O5
def _cam(R=np.eye(3), t=(0, 0, 0), fx=100.0, fy=100.0, cx=50.0, cy=40.0):
    return np.concatenate([np.asarray(R, np.float32).reshape(9), np.asarray(t, np.float32),
                           [fx, fy, cx, cy]]).astype(np.float32)


def test_project_mean_spec_examples():
    cam = _cam()
    m, d, vis = oracle.project_mean(cam, [1, 0, 2])
    assert m[0] == 100.0 and vis and d == 2.0
    m, d, vis = oracle.project_mean(cam, [0, 0, 7])
    assert (m[0], m[1]) == (50.0, 40.0)  # on-axis -> principal point
    assert not oracle.project_mean(cam, [0, 0, -1])[2]  # behind
    assert not oracle.project_mean(cam, [0, 0, 0.005])[2]  # in front of znear but < 0.01


def test_project_mean_rotation_translation():
    # world point projected through a look-at camera equals the pinhole of R mu + t
    cams = sy.orbit_rig(5, 40.0, 320, 200)
    rng = np.random.default_rng(2)
    for c in cams:
        R = c[:9].reshape(3, 3).astype(np.float64)
        t = c[9:12].astype(np.float64)
        for mu in rng.uniform(-1, 1, (20, 3)):
            p = R @ mu + t
            m, d, vis = oracle.project_mean(c, mu)
            assert vis and abs(d - p[2]) < 1e-5
            assert abs(m[0] - (c[12] * p[0] / p[2] + c[14])) < 1e-3
            assert abs(m[1] - (c[13] * p[1] / p[2] + c[15])) < 1e-3


# ------------------------------------------------------------------ O6
def test_cov2d_isotropic_on_axis_closed_form():
    # isotropic sigma on the optical axis at depth z: Sigma2D = diag((fx s/z)^2+0.3, (fy s/z)^2+0.3)
    for sig, z, fx, fy in [(0.1, 2.0, 100.0, 120.0), (0.03, 5.0, 2967.0, 2967.0), (1.0, 10.0, 50.0, 50.0)]:
        cam = _cam(fx=fx, fy=fy, cx=64, cy=48)
        cov, _ = oracle.gaussian_constants(np.array([[1, 0, 0, 0]]), np.array([[sig] * 3]),
                                           np.array([0.5]))
        out, ok = oracle.cov2d(cam, 128, 96, [0, 0, z], cov[0])
        a, b, c, det = out
        ea, ec = (fx * sig / z) ** 2 + 0.3, (fy * sig / z) ** 2 + 0.3
        assert ok and abs(a - ea) <= 2e-6 * ea and abs(c - ec) <= 2e-6 * ec and abs(b) < 1e-6 * ea
        assert abs(det - (a * c - b * b)) <= 1e-6 * det


def test_cov2d_vs_numerical_jacobian():
    # Inside the frustum clamp, Pi_cov = J W Sigma W^T J^T + 0.3 I, with J the Jacobian
    # of the pinhole map p -> (fx px/pz + cx, fy py/pz + cy).  J is obtained here by
    # central differences of the (separately pinned) projection, not from the oracle's formula.
    rng = np.random.default_rng(3)
    cams = sy.orbit_rig(3, 30.0, 320, 200, radius=3.0, height=0.5)
    for c in cams:
        R = c[:9].reshape(3, 3).astype(np.float64)
        t = c[9:12].astype(np.float64)
        fx, fy, cx, cy = [float(v) for v in c[12:]]
        for _ in range(30):
            mu = rng.uniform(-0.5, 0.5, 3)
            q = rng.standard_normal(4)
            s = np.exp(rng.normal(-3, 0.5, 3))
            cov6, _ = oracle.gaussian_constants(q[None], s[None], np.array([0.5]))
            S6 = cov6[0].astype(np.float64)
            Sig = np.array([[S6[0], S6[1], S6[2]], [S6[1], S6[3], S6[4]], [S6[2], S6[4], S6[5]]])
            p = R @ mu + t

            def pi(pp):
                return np.array([fx * pp[0] / pp[2] + cx, fy * pp[1] / pp[2] + cy])

            J = np.zeros((2, 3))
            for a in range(3):
                e = np.zeros(3)
                e[a] = 1e-6 * max(1.0, abs(p[a]))
                J[:, a] = (pi(p + e) - pi(p - e)) / (2 * e[a])
            ref = J @ R @ Sig @ R.T @ J.T + 0.3 * np.eye(2)
            out, ok = oracle.cov2d(c, 320, 200, mu, cov6[0])
            got = np.array([[out[0], out[1]], [out[1], out[2]]])
            assert ok
            assert np.all(np.abs(got - ref) <= 1e-4 * np.max(np.abs(ref)))


def test_cov2d_frustum_clamp_limits_jacobian():
    # far off-axis point: J is evaluated at the clamped point (gsplat classic, O6):
    # Sigma2D must equal the covariance of a point moved onto the clamp boundary
    # at the same depth (the Jacobian then only sees the clamped x/z).
    cam = _cam(fx=100, fy=100, cx=50, cy=40)
    W, H = 100, 80
    cov6, _ = oracle.gaussian_constants(np.array([[1, 0.2, 0.1, 0.3]]), np.array([[0.1, 0.2, 0.05]]),
                                        np.array([0.5]))
    limxp = (W - 50) / 100 + 0.3 * (0.5 * W / 100)
    z = 2.0
    far, _ = oracle.cov2d(cam, W, H, [z * 5.0, 0.1, z], cov6[0])
    edge, _ = oracle.cov2d(cam, W, H, [z * limxp, 0.1, z], cov6[0])
    assert np.allclose(far, edge, rtol=1e-5)


# ------------------------------------------------------------------ O7
def _min_q_over_rect(m, Si, x0, x1, y0, y1):
    """min over the rectangle of (p-m)^T Si (p-m): exact (convex quadratic)."""
    best = np.inf
    if x0 <= m[0] <= x1 and y0 <= m[1] <= y1:
        return 0.0

    def q(x, y):
        d = np.array([x - m[0], y - m[1]])
        return d @ Si @ d

    for (x, fixed_x) in ((x0, True), (x1, True)):  # vertical edges: minimise over y
        yy = m[1] - Si[0, 1] * (x - m[0]) / Si[1, 1]
        best = min(best, q(x, min(max(yy, y0), y1)))
    for y in (y0, y1):
        xx = m[0] - Si[0, 1] * (y - m[1]) / Si[0, 0]
        best = min(best, q(min(max(xx, x0), x1), y))
    return best


def test_accutile_exact_rectangle_test_random_ellipses():
    # A tile is listed iff the ellipse {d^T Sigma^-1 d <= tau} meets the tile's
    # pixel-centre rectangle (O7).  Checked against the exact min of the quadratic
    # form over each rectangle (fp64), with a relative band of 1e-4 for fp32 rounding.
    rng = np.random.default_rng(4)
    TX, TY = 12, 9
    n_checked = 0
    for _ in range(400):
        m = rng.uniform(-20, 16 * TX + 20, 2).astype(np.float32)
        sa, sb = np.exp(rng.uniform(0, 4, 2))
        th = rng.uniform(0, np.pi)
        Rm = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        Sig = Rm @ np.diag([sa ** 2, sb ** 2]) @ Rm.T + 0.3 * np.eye(2)
        a, b, c = np.float32(Sig[0, 0]), np.float32(Sig[0, 1]), np.float32(Sig[1, 1])
        det = np.float32(a * c - b * b)
        tau = np.float32(rng.uniform(0.5, 11.0))
        tiles = set(oracle.tileset(m, (a, b, c, det), tau, TX, TY).tolist())
        S = np.array([[a, b], [b, c]], np.float64)
        Si = np.linalg.inv(S)
        for t in range(TX * TY):
            tx, ty = t % TX, t // TX
            qmin = _min_q_over_rect(m.astype(np.float64), Si, 16 * tx + 0.5, 16 * tx + 15.5,
                                    16 * ty + 0.5, 16 * ty + 15.5)
            if qmin <= tau * (1 - 1e-4):
                assert t in tiles
                n_checked += 1
            elif qmin >= tau * (1 + 1e-4):
                assert t not in tiles
    assert n_checked > 500


def test_accutile_isotropic_closed_form_and_single_tile():
    # single small Gaussian inside one tile -> exactly 1 tile
    t = oracle.tileset(np.array([40.0, 24.0], np.float32), (1.3, 0.0, 1.3, 1.69), 9.0, 10, 10)
    assert t.tolist() == [1 * 10 + 2]
    # isotropic: hit iff the rectangle is within distance ex = sqrt(tau*a) of m
    m = np.array([70.3, 55.1], np.float32)
    a = np.float32(30.0)
    tau = np.float32(4.0)
    tiles = set(oracle.tileset(m, (a, 0.0, a, a * a), tau, 10, 10).tolist())
    r = math.sqrt(float(tau) * float(a))
    for t in range(100):
        tx, ty = t % 10, t // 10
        dx = max(16 * tx + 0.5 - m[0], 0, m[0] - (16 * tx + 15.5))
        dy = max(16 * ty + 0.5 - m[1], 0, m[1] - (16 * ty + 15.5))
        dist = math.hypot(dx, dy)
        if dist < r * (1 - 1e-5):
            assert t in tiles
        elif dist > r * (1 + 1e-5):
            assert t not in tiles


def test_accutile_far_offscreen_is_empty_and_huge_is_clamped():
    assert oracle.tileset(np.array([-1e6, 5.0], np.float32), (2, 0, 2, 4), 9.0, 8, 8).size == 0
    t = oracle.tileset(np.array([60.0, 60.0], np.float32), (1e8, 0, 1e8, 1e16), 9.0, 8, 8)
    assert t.size == 64  # covers the whole 8x8 grid, nothing out of range


# ------------------------------------------------------------------ O9
def test_key_layout_spec_example():
    ex = GOLD["keys"][0]
    dbits = struct.unpack("<I", struct.pack("<f", ex["depth"]))[0]
    key = (ex["t"] << (32 + ex["bitK"])) | (ex["k"] << 32) | dbits
    assert key == ex["expect"] == eval(ex["expect_formula"])
    # positive floats: raw-bit order == numeric order
    d = np.sort(np.float32(np.random.default_rng(0).uniform(0.01, 100, 1000)))
    assert np.all(np.diff(d.view(np.uint32).astype(np.int64)) >= 0)
