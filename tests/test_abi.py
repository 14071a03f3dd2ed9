"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports
every symbol include/coherent_raster.h declares; the binding's structs match
the header layout; the product package never imports the oracle."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "coherent_raster.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2605_04509_b200 import build, _native
    path = build.build()
    return _native.load(path)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cr_[a-z_]+)\s*\(", src)))


def test_header_declares_binding_symbols():
    from paper_2605_04509_b200 import _native
    assert sorted(_native.SYMBOLS) == declared_functions()


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_version_and_status_strings(lib):
    assert lib.cr_version().decode().startswith("coherent_raster sm_100a")
    assert lib.cr_status_string(4) == b"CR_ERR_TILE_ID_OVERFLOW"


def test_struct_layouts(tmp_path):
    # compare ctypes layouts with what the C compiler makes of the header
    from paper_2605_04509_b200 import _native as N
    src = tmp_path / "l.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "coherent_raster.h"\n'
        'int main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(cr_camera), '
        'sizeof(cr_display), offsetof(cr_display, lens_pitch), sizeof(cr_render_opts), '
        'offsetof(cr_render_opts, background), sizeof(cr_stats), '
        'offsetof(cr_stats, ms_preprocess), offsetof(cr_stats, device_bytes));return 0;}\n')
    exe = tmp_path / "l"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    exp = [C.sizeof(N.Camera), C.sizeof(N.Display), N.Display.lens_pitch.offset,
           C.sizeof(N.RenderOpts), N.RenderOpts.background.offset, C.sizeof(N.Stats),
           N.Stats.ms_preprocess.offset, N.Stats.device_bytes.offset]
    assert got == exp


def test_orbit_rig_helper_matches_synthetic(lib):
    # the ABI's host helper builds the same rig as the seeded input module
    import numpy as np
    from paper_2605_04509_b200 import synthetic as sy
    from paper_2605_04509_b200.raster import CoherentRaster
    c = sy.CONFIGS["C"]
    a = CoherentRaster.make_orbit_rig(c.display(), radius=4.0, height=0.8, fov_y_deg=40.0)
    b = c.make_rig()
    assert np.allclose(a, b, atol=2e-5 * np.abs(b).max())


def test_no_cuda_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_04509_b200._native import CrError
    from paper_2605_04509_b200.raster import CoherentRaster
    with pytest.raises((CrError, RuntimeError, AssertionError)):
        CoherentRaster(0)


def test_product_package_does_not_reference_oracle():
    pkg = os.path.join(ROOT, "paper_2605_04509_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "liboracle" not in txt and "oracle.cpp" not in txt, f
