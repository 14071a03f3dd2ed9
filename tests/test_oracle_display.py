"""Pins for the oracle's display model: O1 view map (Eqs.1-3) and
O2 remap table Psi (Eq.8).  CPU only."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _vmap(W, H, N, Lx, tan_alpha, Koff):
    o = oracle.Oracle(nthreads=2)
    o.set_display(W, H, N, Lx, tan_alpha=tan_alpha, center_offset=Koff)
    return o.view_map()


@pytest.mark.parametrize("ex", GOLD["view_map"])
def test_view_map_spec_examples(ex):
    V = _vmap(ex["W"], ex["H"], ex["N"], ex["Lx"], ex["tan_alpha"], ex["Koff"])
    for x, y, u, j in ex.get("expect", []):
        assert V[y, x, u] == j, ex["cite"]
    if "expect_row0" in ex:
        assert list(V[0].reshape(-1)) == ex["expect_row0"], ex["cite"]


def _exact_j(x, y, u, N, Lx, tA, K):
    """Eqs.1-3 in exact rational arithmetic (the plain definition)."""
    d = Fraction(3 * x + u) + Fraction(3 * y) * Fraction(tA) - Fraction(K)
    L = Fraction(Lx)
    xo = d - L * math.floor(d / L)
    return min(max(math.floor(N * xo / L), 0), N - 1)


def test_view_map_equals_exact_rational_on_dyadic_display():
    # dyadic Lx, tan(alpha), K_offset: every fp64 op is exact, so the oracle
    # must equal the exact rational evaluation of Eqs.1-3 everywhere.
    W, H, N, Lx, tA, K = 53, 37, 7, 12.5, 0.25, 1.5
    V = _vmap(W, H, N, Lx, tA, K)
    for y in range(H):
        for x in range(W):
            for u in range(3):
                assert V[y, x, u] == _exact_j(x, y, u, N, Lx, tA, K)


def test_view_map_vs_exact_rational_general_display():
    # Looking-Glass-like parameters: fp64 may only differ from exact arithmetic
    # where N*x_off/Lx is within rounding of an integer (a view boundary).
    W, H, N, Lx, tA, K = 97, 61, 100, 19.6153, 0.1852, 7.3
    V = _vmap(W, H, N, Lx, tA, K)
    bad = 0
    for y in range(0, H, 3):
        for x in range(W):
            for u in range(3):
                j = _exact_j(x, y, u, N, Lx, tA, K)
                if V[y, x, u] != j:
                    d = Fraction(3 * x + u) + Fraction(3 * y) * Fraction(tA) - Fraction(K)
                    L = Fraction(Lx)
                    v = N * (d - L * math.floor(d / L)) / L
                    assert abs(v - round(v)) < Fraction(1, 10 ** 9)
                    bad += 1
    assert bad <= 2


def test_view_map_range_and_uniformity():
    W, H, N = 480, 270, 100
    V = _vmap(W, H, N, 19.6153, 0.1852, 7.3)
    assert V.max() < N
    share = np.bincount(V.reshape(-1), minlength=N) / V.size
    # each view occupies Lx/N of every lens period -> share 1/N (+- edge effects)
    assert np.all(np.abs(share * N - 1.0) < 0.05)


def test_view_map_periodicity_alpha0():
    # alpha = 0, integer Lx: V periodic in the subpixel linearisation 3x+u with period Lx
    W, H, N, Lx = 40, 3, 4, 10
    V = _vmap(W, H, N, float(Lx), 0.0, 2.0)
    lin = V.reshape(H, W * 3)
    assert np.array_equal(lin[:, Lx:], lin[:, :-Lx])
    # alpha = 0 -> every row identical
    assert np.array_equal(lin[0], lin[1]) and np.array_equal(lin[1], lin[2])


def test_view_map_slant_invariant():
    # tan(alpha) = 0.5, dyadic Lx/K: moving 2 rows down shifts d by exactly 3 = one pixel,
    # so V(x, y+2, u) == V(x+1, y, u) exactly (SURVEY §8c pins, checked here).
    W, H = 200, 100
    V = _vmap(W, H, 9, 12.5, 0.5, 1.5)
    assert np.array_equal(V[2:, :-1, :], V[:-2, 1:, :])


def test_view_map_mask_channel():
    # Lx=3, alpha=0, N=3: the mask for j=0 selects exactly channel u=0
    V = _vmap(17, 5, 3, 3.0, 0.0, 0.0)
    assert np.all((V == 0) == (np.arange(3)[None, None, :] == 0))


def test_view_map_negative_offset_floor_mod():
    # K_offset larger than 3x+u -> negative d_offset; floor-mod lands in [0,Lx)
    V = _vmap(4, 1, 4, 8.0, 0.0, 30.0)
    for x in range(4):
        for u in range(3):
            d = 3 * x + u - 30
            assert V[0, x, u] == math.floor(4 * (d % 8) / 8)


# ------------------------------------------------------------------- O2: Psi
def _psi_props(V, psi, remap):
    H, W, _ = V.shape
    TX, TY = (W + 15) // 16, (H + 15) // 16
    for t in range(TX * TY):
        tx, ty = t % TX, t // TX
        nx, ny = min(16, W - 16 * tx), min(16, H - 16 * ty)
        n = nx * ny * 3
        row = psi[t]
        assert np.all(row[n:] == 0xFFFF)
        ell = row[:n].astype(np.int64)
        valid = sorted((ly * 16 + lx) * 3 + u for ly in range(ny) for lx in range(nx) for u in range(3))
        assert sorted(ell.tolist()) == valid  # bijection on the tile's subpixels
        ly, rem = ell // 48, ell % 48
        vals = V[16 * ty + ly, 16 * tx + rem // 3, rem % 3].astype(np.int64)
        if remap:
            assert np.all(np.diff(vals) >= 0)  # Eq.8 monotonicity
            same = np.diff(vals) == 0
            assert np.all(np.diff(ell)[same] > 0)  # stable (row-major ties)
        else:
            assert np.array_equal(ell, np.array(valid))


def test_remap_properties_random_configs():
    # SPEC acceptance 4: 50 random displays, every tile a bijection + monotone
    rng = np.random.default_rng(5)
    for it in range(50):
        W, H = int(rng.integers(1, 70)), int(rng.integers(1, 40))
        a = math.radians(rng.uniform(-15, 15))
        Lx = float(rng.uniform(2, 40))
        K = float(rng.uniform(-Lx, Lx))
        N = int(rng.integers(1, 65))
        o = oracle.Oracle(nthreads=2)
        o.set_display(W, H, N, Lx, slant=a, center_offset=K)
        V = o.view_map()
        _psi_props(V, o.remap(1), True)
        if it < 5:
            _psi_props(V, o.remap(0), False)


def test_remap_single_view_identity():
    o = oracle.Oracle(nthreads=2)
    o.set_display(40, 20, 1, 5.0, slant=0.2, center_offset=0.3)
    assert np.array_equal(o.remap(1), o.remap(0))
