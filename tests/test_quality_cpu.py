"""N2 reuse-quality harness, CPU pins: the harness's SSIM / PSNR against an
independent scipy implementation of the same definitions (Wang et al. SSIM
with the 3DGS evaluation convention: Gaussian window 11, sigma 1.5, zero
padding, C1 = 0.01^2, C2 = 0.03^2), and the oracle's per-view frames
 interlacing exactly to its subpixel image (Eq.4)."""
import math

import numpy as np
import torch
from scipy import ndimage

import oracle
from paper_2605_04509_b200 import quality, synthetic as sy


def _ssim_scipy(a, b):
    x = np.arange(11) - 5
    g = np.exp(-x * x / (2 * 1.5 ** 2))
    g /= g.sum()
    w = np.outer(g, g)
    vals = []
    for ch in range(3):
        p, q = a[..., ch].astype(np.float64), b[..., ch].astype(np.float64)
        f = lambda z: ndimage.correlate(z, w, mode="constant", cval=0.0)  # noqa: E731
        mp, mq = f(p), f(q)
        spp, sqq, spq = f(p * p) - mp * mp, f(q * q) - mq * mq, f(p * q) - mp * mq
        c1, c2 = 0.01 ** 2, 0.03 ** 2
        vals.append(((2 * mp * mq + c1) * (2 * spq + c2)) /
                    ((mp * mp + mq * mq + c1) * (spp + sqq + c2)))
    return float(np.mean(vals))


def test_ssim_matches_independent_scipy_implementation():
    rng = np.random.default_rng(0)
    a = rng.random((3, 40, 56, 3))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    got = quality.ssim_per_image(torch.from_numpy(a), torch.from_numpy(b)).numpy()
    ref = np.array([_ssim_scipy(a[i], b[i]) for i in range(3)])
    assert np.allclose(got, ref, atol=1e-10)
    assert np.allclose(quality.ssim_per_image(torch.from_numpy(a), torch.from_numpy(a)).numpy(), 1.0)
    assert np.all(got < 1.0) and np.all(got > 0.5)


def test_psnr_closed_form():
    a = torch.zeros(2, 8, 8, 3, dtype=torch.float64)
    b = a.clone()
    b[0] += 0.1  # mse 0.01 -> 20 dB
    p = quality.psnr_per_image(b, a)
    assert abs(float(p[0]) - 20.0) < 1e-9 and math.isinf(float(p[1]))


def test_oracle_view_frames_interlace_to_the_subpixel_image():
    # Eq.4 picks view V[y][x][u] per subpixel: interlacing the per-view frames of
    # the same render reproduces the subpixel image exactly (same lists and ops)
    c = sy.CONFIGS["A"]
    o = oracle.Oracle(nthreads=4)
    o.set_scene(c.make_scene())
    o.set_display(c.W, c.H, c.N, c.lens_pitch, slant=c.slant, center_offset=c.center_offset)
    o.set_rig(c.make_rig())
    for s in (1, 4):
        o.render(s=s, bg=(0.1, 0.0, 0.3))
        F = o.view_frames()
        V = o.view_map()
        y, x, u = np.indices(V.shape)
        assert np.array_equal(F[V, y, x, u], o.image())
