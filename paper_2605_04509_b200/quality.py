"""Reuse-quality harness (the paper's T1 evaluation).

The paper measures PSNR, SSIM and LPIPS "on per-view images" against images
rendered by the original 3DGS as pseudo ground truth.  Here:

* per-view images at cluster size s: every view j rendered full frame with
  the shared attributes of its cluster (the library's CR_FLAG_VIEW_FRAMES path:
  the same lists, means and blend arithmetic as the interlaced render, which
  they reproduce exactly when interlaced);
* pseudo ground truth: the same at s = 1 (every view with its own
  attributes — plain per-view 3DGS);
* PSNR per view on [0,1]-clamped float images; SSIM per view with the 3DGS
  evaluation convention (Gaussian window 11, sigma 1.5, zero-padded 'same'
  filtering, C1 = 0.01^2, C2 = 0.03^2, mean over channels and pixels);
* LPIPS is out of scope (needs trained network weights).

Metric arithmetic runs in PyTorch on the GPU (this is a measurement tool, not
the hot path).  CLI: python -m paper_2605_04509_b200.quality C 2,4,8,10,16
"""
from __future__ import annotations

import math
import sys

import torch
import torch.nn.functional as F

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


def _gauss_window(device, dtype):
    x = torch.arange(SSIM_WINDOW, device=device, dtype=dtype) - SSIM_WINDOW // 2
    g = torch.exp(-(x * x) / (2 * SSIM_SIGMA ** 2))
    g = g / g.sum()
    return g


def _blur(x, g):
    """Separable zero-padded 'same' Gaussian filter of [B, C, H, W]."""
    C = x.shape[1]
    p = SSIM_WINDOW // 2
    x = F.conv2d(x, g.view(1, 1, 1, -1).expand(C, 1, 1, -1), padding=(0, p), groups=C)
    return F.conv2d(x, g.view(1, 1, -1, 1).expand(C, 1, -1, 1), padding=(p, 0), groups=C)


def ssim_per_image(a: torch.Tensor, b: torch.Tensor, chunk: int = 4) -> torch.Tensor:
    """SSIM of each image pair; a, b: [B, H, W, 3] in [0, 1].  Returns [B] (float64)."""
    out = []
    for q in range(0, a.shape[0], chunk):
        x = a[q:q + chunk].permute(0, 3, 1, 2).double()
        y = b[q:q + chunk].permute(0, 3, 1, 2).double()
        g = _gauss_window(x.device, x.dtype)
        mx, my = _blur(x, g), _blur(y, g)
        sxx = _blur(x * x, g) - mx * mx
        syy = _blur(y * y, g) - my * my
        sxy = _blur(x * y, g) - mx * my
        m = ((2 * mx * my + SSIM_C1) * (2 * sxy + SSIM_C2)) / \
            ((mx * mx + my * my + SSIM_C1) * (sxx + syy + SSIM_C2))
        out.append(m.mean(dim=(1, 2, 3)))
    return torch.cat(out)


def psnr_per_image(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """PSNR (dB, peak 1) of each image pair; [B, H, W, 3] -> [B] (inf where equal)."""
    mse = ((a.double() - b.double()) ** 2).mean(dim=(1, 2, 3))
    return 10 * torch.log10(1.0 / mse)


def view_frames(r, s: int) -> torch.Tensor:
    """Per-view frames [N, H, W, 3] (float, clamped to [0, 1]) at cluster size s."""
    return r.render(s, output_format="float", view_frames=True).clamp_(0.0, 1.0)


def reuse_quality(r, s_list, timing_frames: int = 3):
    """Per-view PSNR / SSIM of cluster sizes s_list against s = 1 (pseudo GT),
    plus the interlaced-image PSNR and the interlaced frame time of each s."""
    ref = view_frames(r, 1)
    ref_il = r.render(1, output_format="float").clamp(0, 1)
    rows = []
    for s in s_list:
        for _ in range(2):
            r.render(s, stats=True)
        ms = sorted((r.render(s, stats=True), r.last_stats["ms_total"])[1]
                    for _ in range(timing_frames))[timing_frames // 2]
        pairs = r.last_stats["pairs"]
        K = r.last_stats["num_clusters"]
        fr = view_frames(r, s)
        pv = psnr_per_image(fr, ref)
        sv = ssim_per_image(fr, ref)
        il = r.render(s, output_format="float").clamp(0, 1)
        mse = float(((il.double() - ref_il.double()) ** 2).mean())
        fin = pv[torch.isfinite(pv)]
        rows.append(dict(s=s, K=K, pairs=pairs, frame_ms=ms,
                         psnr_interlaced=(10 * math.log10(1 / mse) if mse > 0 else math.inf),
                         psnr_view_mean=float(fin.mean()) if fin.numel() else math.inf,
                         psnr_view_min=float(pv.min()),
                         ssim_view_mean=float(sv.mean()), ssim_view_min=float(sv.min()),
                         psnr_views=pv.cpu().tolist(), ssim_views=sv.cpu().tolist()))
        del fr
    return rows


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    from . import CoherentRaster
    from . import synthetic as sy
    name = argv[0] if argv else "C"
    s_list = [int(v) for v in (argv[1] if len(argv) > 1 else "2,4,8,10,16").split(",")]
    c = sy.CONFIGS[name]
    r = CoherentRaster(0)
    r.upload_gaussians(c.make_scene())
    r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
    r.set_camera_rig(c.make_rig())
    print(f"config {name}: {c.M} Gaussians SH{c.sh_degree}, {c.N} views, {c.W}x{c.H}; "
          "pseudo ground truth = per-view frames at s = 1 (P:478-480)")
    print("| s | K | pairs | frame ms | interlaced PSNR | per-view PSNR mean / min (dB) "
          "| per-view SSIM mean / min |")
    print("|---|---|---|---|---|---|---|")
    for row in reuse_quality(r, s_list):
        print(f"| {row['s']} | {row['K']} | {row['pairs']} | {row['frame_ms']:.2f} | "
              f"{row['psnr_interlaced']:.2f} | {row['psnr_view_mean']:.2f} / "
              f"{row['psnr_view_min']:.2f} | {row['ssim_view_mean']:.4f} / "
              f"{row['ssim_view_min']:.4f} |", flush=True)


if __name__ == "__main__":
    main()
