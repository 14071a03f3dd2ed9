"""Per-rank cost of the row-band split measured on one GPU: render band r of R
(the work one rank does) and report stage times.  python tools/band_cost.py C 8"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
from paper_2605_04509_b200.multigpu import band_rows, balanced_bands, row_pair_weights
name = sys.argv[1]; R = int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "equal"
c = sy.CONFIGS[name]
r = CoherentRaster(0)
r.upload_gaussians(c.make_scene())
r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
r.set_camera_rig(c.make_rig())
worst = 0
bands = None
if mode in ("balanced", "refined"):
    r.render(c.cluster_size)
    torch.cuda.synchronize()
    wrow = row_pair_weights(r, c.cluster_size) + 2.0e5
    bands = balanced_bands(wrow, R)
    if mode == "refined":  # the bench's measured-cost refinement, simulated on one GPU
        from paper_2605_04509_b200.multigpu import refine_bands
        for _ in range(2):
            costs = []
            for q in range(R):
                cs = []
                for _ in range(3):
                    r.render(c.cluster_size, rows=bands[q], stats=True)
                    cs.append(r.last_stats["ms_total"] - r.last_stats["ms_preprocess"])
                costs.append(min(cs))
            bands, wrow = refine_bands(wrow, bands, costs, R)
for q in range(R):
    rows = bands[q] if bands else band_rows(r.TY, R, q)
    for _ in range(2):
        r.render(c.cluster_size, rows=rows, stats=True)
    ms = []
    for _ in range(5):
        r.render(c.cluster_size, rows=rows, stats=True)
        ms.append(r.last_stats["ms_total"])
    st = r.last_stats
    ms.sort()
    worst = max(worst, ms[2])
    print(f"band {q}/{R} rows {rows}: total {ms[2]:.2f} ms pre {st['ms_preprocess']:.2f} bin {st['ms_bin']:.2f} sort {st['ms_sort']:.2f} comp {st['ms_composite']:.2f} pairs {st['pairs']}", flush=True)
print(f"R={R}: slowest band {worst:.2f} ms -> {1000/worst:.1f} frames/s (before the all-gather)")
