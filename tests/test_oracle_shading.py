"""Pins for the oracle's shading: O11 SH colour (Eq.6 Pi_SH) and O12
compositing (Eqs.9-10).  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import sph_harm_y

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _dirs(n, seed=0):
    d = np.random.default_rng(seed).standard_normal((n, 3))
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def test_sh_spec_examples():
    sh = np.zeros((1, 3), np.float32)
    sh[0] = 0.7
    for d in _dirs(5):
        rgb = oracle.eval_sh(0, sh, d)
        assert np.allclose(rgb, 0.28209479177 * np.float32(0.7) + 0.5, atol=1e-9)
    z = np.zeros((16, 3), np.float32)
    assert np.allclose(oracle.eval_sh(3, z, _dirs(1)[0]), 0.5)
    c = np.zeros((4, 3), np.float32)
    c[3] = 0.4  # the l=1 band coefficient that multiplies x
    diff = oracle.eval_sh(1, c, np.array([1.0, 0, 0])) - oracle.eval_sh(1, c, np.array([-1.0, 0, 0]))
    assert np.allclose(np.abs(diff), 2 * 0.48860251190 * np.float32(0.4), rtol=1e-9)


def _real_sh(l, m, d):
    """Real spherical harmonics from scipy's complex Y_l^m (independent routine)."""
    theta = np.arccos(np.clip(d[:, 2], -1, 1))  # polar from +z
    phi = np.arctan2(d[:, 1], d[:, 0])
    if m == 0:
        return np.real(sph_harm_y(l, 0, theta, phi))
    Y = sph_harm_y(l, abs(m), theta, phi)
    if m > 0:
        return math.sqrt(2) * (-1) ** m * np.real(Y)
    return math.sqrt(2) * (-1) ** m * np.imag(Y)


def test_sh_basis_matches_real_spherical_harmonics():
    # Each 3DGS basis function (index l^2 + l + m, ordered m=-l..l) must equal the
    # textbook real SH Y_lm up to one fixed sign per function (the 3DGS sign
    # convention), over many directions.  Catches dropped terms, wrong constants
    # and transposed axes.
    D = _dirs(200, seed=1)
    B = np.stack([oracle.sh_basis(3, d) for d in D])
    for l in range(4):
        for m in range(-l, l + 1):
            idx = l * l + l + m
            ref = _real_sh(l, m, D)
            sgn = np.sign(np.sum(B[:, idx] * ref))
            assert sgn != 0
            assert np.allclose(B[:, idx], sgn * ref, atol=1e-12), (l, m)


def test_sh_linearity():
    rng = np.random.default_rng(2)
    c = rng.standard_normal((16, 3)).astype(np.float32)
    for d in _dirs(10, 3):
        base = oracle.eval_sh(3, c, d) - 0.5
        assert np.allclose(oracle.eval_sh(3, (2 * c).astype(np.float32), d) - 0.5, 2 * base,
                           atol=1e-12)


# ------------------------------------------------------------------- O12
@pytest.mark.parametrize("ex", GOLD["blend"])
def test_blend_spec_examples(ex):
    s = np.array(ex["splats"], np.float32).reshape(-1, 7)
    assert oracle.blend(s, ex["px"], ex["py"], ex["bg"]) == pytest.approx(ex["expect"], abs=1e-7)


def test_blend_single_isotropic_closed_form():
    # C(p) = c*alpha(p) + bg*(1-alpha(p)), alpha = min(0.99, o exp(-|p-m|^2/(2 s2)))
    # when alpha >= 1/255, else C = bg (Eqs.9-10 with one Gaussian)
    s2, o, col, bg = 9.0, 0.8, 0.9, 0.2
    m = (10.0, 7.0)
    for px in np.linspace(0.5, 25.5, 26):
        for py in (7.5, 9.5, 12.5):
            r2 = (px - m[0]) ** 2 + (py - m[1]) ** 2
            a = min(0.99, o * math.exp(-r2 / (2 * s2)))
            exp = col * a + bg * (1 - a) if a >= 1 / 255 else bg
            splat = np.array([[m[0], m[1], 1 / s2, 0, 1 / s2, o, col]], np.float32)
            assert oracle.blend(splat, px, py, bg) == pytest.approx(exp, abs=2e-6)


def test_blend_saturation_stops_before_blending():
    # n coincident opaque splats (alpha = 0.99 clamp): T = 0.01 after one, 1e-4 would be
    # reached by the second -> stop before blending it (T(1-a) < 1e-4).
    s = np.array([[0, 0, 1, 0, 1, 1.0, 1.0]] * 3, np.float32)
    v = oracle.blend(s, 0.0, 0.0, 0.0)
    assert v == pytest.approx(0.99, abs=1e-6)
    # below 1/255 is skipped entirely
    s = np.array([[0, 0, 1, 0, 1, 1.0 / 256, 1.0]], np.float32)
    assert oracle.blend(s, 0.0, 0.0, 0.5) == 0.5


def test_blend_geometric_series():
    # n coincident splats with alpha a: C = sum_{e<n} a(1-a)^e while T stays >= 1e-4
    a = 0.3
    for n in range(1, 12):
        s = np.array([[0, 0, 1, 0, 1, a, 1.0]] * n, np.float32)
        exp = sum(a * (1 - a) ** e for e in range(n))
        assert oracle.blend(s, 0.0, 0.0, 0.0) == pytest.approx(exp, abs=5e-6)
