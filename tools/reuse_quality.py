"""SURVEY N2 / paper T1 analogue: image quality of Cross-view Coherent Attribute
Reuse against exact per-view attributes (s=1) on a synthetic scene, with the
frame time of each s.  python tools/reuse_quality.py C 1,2,4,8,10,16"""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
name = sys.argv[1] if len(sys.argv) > 1 else "C"
ss = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,10,16").split(",")]
c = sy.CONFIGS[name]
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
V = torch.from_numpy(r.view_map().astype(np.int64)).cuda()
ref = r.render(1, output_format="float").clamp(0, 1).double()
print(f"config {name}: {c.M} Gaussians, {c.N} views, {c.W}x{c.H}")
print("| s | K | pairs | frame ms | PSNR interlaced (dB) | mean per-view PSNR (dB) | min per-view PSNR (dB) |")
print("|---|---|---|---|---|---|---|")
for s in ss:
    for _ in range(2):
        r.render(s, stats=True)
    ms = sorted((r.render(s, stats=True), r.last_stats["ms_total"])[1] for _ in range(3))[1]
    pairs = r.last_stats["pairs"]
    img = r.render(s, output_format="float").clamp(0, 1).double()
    err = (img - ref) ** 2
    mse = err.mean().item()
    ps = 10 * math.log10(1 / mse) if mse > 0 else float("inf")
    # per-view (deinterlaced, masked) PSNR
    sums = torch.zeros(c.N, dtype=torch.float64, device="cuda").index_add_(0, V.reshape(-1), err.reshape(-1))
    cnts = torch.bincount(V.reshape(-1), minlength=c.N).double()
    pv = (10 * torch.log10(cnts / sums.clamp_min(1e-30))).cpu().numpy()
    pv = np.where(np.isfinite(pv), pv, np.inf)
    fin = pv[np.isfinite(pv)]
    print(f"| {s} | {-(-c.N // s)} | {pairs} | {ms:.2f} | {ps:.2f} | {fin.mean() if fin.size else float('inf'):.2f} | {fin.min() if fin.size else float('inf'):.2f} |", flush=True)
