"""GPU parity on randomised small configurations: ragged panels, view counts
N in [1, 60], cluster sizes s in [1, min(N, 32)], lens pitch / slant / offset
(Eqs.1-3), SH degree 0-3, camera arcs from a single pose to wide
cones, near planes cutting the scene, background colours and tile-row bands —
each against the CPU oracle: view map and Psi, sorted keys and payloads,
ranges and per-record counts bit-exact; images within 2/255 and >= 50 dB
(check_frame).  Seeds are fixed, so every case is reproducible."""
import numpy as np
import pytest

from paper_2605_04509_b200 import synthetic as sy
from test_gpu_parity import _need_gpu, check_frame, make_pair

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    W = int(rng.integers(40, 420))
    H = int(rng.integers(24, 260))
    N = int(rng.integers(1, 61))
    s = int(rng.integers(1, min(N, 32) + 1))
    Lx = float(rng.uniform(3.0, 40.0))
    slant = float(rng.uniform(-0.6, 0.6))
    Koff = float(rng.uniform(-20.0, 20.0))
    deg = int(rng.integers(0, 4))
    M = int(rng.integers(500, 4000))
    sc = sy.random_scene(M, deg, seed=seed, scale_median=float(rng.uniform(0.01, 0.12)))
    cone = float(rng.choice([0.0, rng.uniform(0.5, 10.0), rng.uniform(10.0, 60.0)]))
    cams = sy.orbit_rig(N, cone, W, H, radius=float(rng.uniform(2.0, 4.0)),
                        height=float(rng.uniform(-0.5, 1.0)), fov_y_deg=float(rng.uniform(30.0, 70.0)))
    znear = float(rng.choice([0.01, rng.uniform(1.0, 2.5)]))
    bg = tuple(float(v) for v in rng.uniform(0.0, 0.5, 3))
    TY = (H + 15) // 16
    r0 = int(rng.integers(0, TY))
    rows = (r0, int(rng.integers(r0 + 1, TY + 1)))
    return sc, W, H, N, s, Lx, slant, Koff, cams, znear, bg, rows


@pytest.mark.parametrize("seed", range(40))
def test_random_configuration(seed):
    _need_gpu()
    sc, W, H, N, s, Lx, slant, Koff, cams, znear, bg, rows = _case(seed)
    g, o = make_pair(sc, W, H, N, Lx, slant, Koff, cams, znear=znear)
    assert np.array_equal(g.view_map(), o.view_map())
    assert np.array_equal(g.remap_table().reshape(-1), o.remap(1).reshape(-1))
    check_frame(g, o, s, bg=bg)
    check_frame(g, o, s, rows=rows, bg=bg)
