"""N4: PLY ingestion of trained-3DGS scenes."""
import numpy as np
import pytest

from paper_2605_04509_b200 import ply, synthetic as sy


@pytest.mark.parametrize("deg", [0, 1, 3])
def test_round_trip(deg):
    sc = sy.random_scene(500, deg, seed=deg)
    back = ply.load_ply(ply.save_ply(sc))
    assert back["sh_degree"] == deg
    for k in ("means", "quats", "sh"):
        assert np.array_equal(back[k], sc[k]), k
    assert np.allclose(back["scales"], sc["scales"], rtol=1e-6)
    assert np.allclose(back["opacities"], sc["opacities"], atol=1e-6)


def test_activations_and_errors():
    sc = sy.random_scene(1, 0, 0)
    sc["opacities"][:] = 0.5  # logit 0 -> 0.5
    sc["scales"][:] = 1.0     # log-scale 0 -> 1
    back = ply.load_ply(ply.save_ply(sc))
    assert back["opacities"][0] == pytest.approx(0.5) and np.all(back["scales"] == 1.0)
    with pytest.raises(ply.PlyError, match="MalformedHeader"):
        ply.load_ply(b"not a ply")
    blob = ply.save_ply(sy.random_scene(10, 0, 0))
    with pytest.raises(ply.PlyError, match="TruncatedBody"):
        ply.load_ply(blob[:-8])
    with pytest.raises(ply.PlyError, match="UnsupportedFormat"):
        ply.load_ply(blob.replace(b"binary_little_endian", b"ascii"))


def test_header_property_order_is_inria():
    # INRIA 3DGS vertex layout: x y z, f_dc_0..2, f_rest_*, opacity,
    # scale_0..2, rot_0..3 — tools that read by position expect exactly this order.
    blob = ply.save_ply(sy.random_scene(3, 1, 0))
    head = blob[:blob.index(b"end_header")].decode().splitlines()
    props = [ln.split()[-1] for ln in head if ln.startswith("property")]
    rest = [f"f_rest_{i}" for i in range(9)]
    assert props == (["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"] + rest + ["opacity"]
                     + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)])
