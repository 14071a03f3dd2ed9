"""N2 reuse-quality harness on the GPU against the oracle (config A):
per-view frames (CR_FLAG_VIEW_FRAMES) within the image tolerance of the
oracle's per-view frames, interlacing exactly to the subpixel render, and the
harness's per-view PSNR / SSIM of s = 4 against s = 1 equal to the values the
oracle's frames give (0.01 dB, 1e-4)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_04509_b200 import quality, synthetic as sy
from test_gpu_parity import _need_gpu, psnr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pairA():
    _need_gpu()
    from paper_2605_04509_b200 import CoherentRaster
    c = sy.CONFIGS["A"]
    sc, cams = c.make_scene(), c.make_rig()
    g = CoherentRaster(0)
    g.upload_gaussians(sc)
    g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset)
    g.set_camera_rig(cams)
    o = oracle.Oracle()
    o.set_scene(sc)
    o.set_display(c.W, c.H, c.N, c.lens_pitch, slant=c.slant, center_offset=c.center_offset)
    o.set_rig(cams)
    return g, o, c


@pytest.mark.parametrize("s", [1, 4])
def test_view_frames_match_oracle_and_interlace(pairA, s):
    g, o, c = pairA
    fr = g.render(s, output_format="float", view_frames=True).cpu().numpy()
    assert fr.shape == (c.N, c.H, c.W, 3)
    o.render(s=s)
    ref = o.view_frames()
    assert np.abs(fr - ref).max() <= 2 / 255
    assert psnr(np.clip(fr, 0, 1), np.clip(ref, 0, 1)) >= 50
    V = g.view_map()
    y, x, u = np.indices(V.shape)
    il = g.render(s, output_format="float").cpu().numpy()
    assert np.array_equal(fr[V, y, x, u], il)
    fr8 = g.render(s, view_frames=True).cpu().numpy()
    assert fr8.dtype == np.uint8 and np.abs(fr8.astype(int) - oracle.quantize_rgb8(ref)).max() <= 2


def test_reuse_quality_harness_matches_oracle(pairA):
    # per-view PSNR and SSIM of s=4 against s=1 pseudo ground truth
    g, o, c = pairA
    row = quality.reuse_quality(g, [4], timing_frames=1)[0]
    o.render(s=1)
    ref = np.clip(o.view_frames(), 0, 1)
    o.render(s=4)
    got = np.clip(o.view_frames(), 0, 1)
    pv = quality.psnr_per_image(torch.from_numpy(got), torch.from_numpy(ref)).numpy()
    sv = quality.ssim_per_image(torch.from_numpy(got), torch.from_numpy(ref)).numpy()
    fin = np.isfinite(pv)
    assert np.allclose(np.asarray(row["psnr_views"])[fin], pv[fin], atol=0.01)
    assert np.allclose(row["ssim_views"], sv, atol=1e-4)
    assert 25 < row["psnr_view_mean"] < np.inf and 0.9 < row["ssim_view_mean"] < 1.0
