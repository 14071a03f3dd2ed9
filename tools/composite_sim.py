#!/usr/bin/env python
"""Composite work-schedule simulator (design exploration, not a test).

Uses the CPU oracle's per-(i,k) records and sorted (t,k) lists on sampled
tiles of a config to count, per candidate warp schedule of the a9 composite,
the warp-level blend-loop iterations and staging batches — the quantities that
set the composite's issue time.  Schedules:
  A   chunks of 32 Psi ranks, per 32-entry batch per-view box masks, each
      lane walks its view's mask (round-1 k_composite_staged)
  VL  same chunks, per-view compacted lists over super-batches of SB entries
  P2  chunks of up to 64 ranks, two consecutive ranks per lane, lane walks the
      union of its two views' masks (per 32-entry batch)
usage: python tools/composite_sim.py [config] [ntiles]
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2605_04509_b200 import synthetic as sy  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C"
    ntiles = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    c = sy.CONFIGS[name]
    scene, cams = c.make_scene(), c.make_rig()
    o = oracle.Oracle()
    o.set_scene(scene)
    o.set_display(c.W, c.H, c.N, c.lens_pitch, slant=c.slant, center_offset=c.center_offset)
    o.set_rig(cams)
    TX, TY = (c.W + 15) // 16, (c.H + 15) // 16
    rng = np.random.default_rng(5)
    tiles = np.unique(rng.choice(TX * TY, ntiles, replace=False)).astype(np.int32)
    s = c.cluster_size
    o.render(s=s, tiles=tiles, composite=False)
    keys, pay = o.pairs()
    S, E = o.ranges()
    rec = o.records()
    _, tau = o.constants()
    V = o.view_map()
    psi = o.remap(1)
    K = o.K
    R = cams[:, :9].reshape(-1, 3, 3).astype(np.float64)
    tv = cams[:, 9:12].astype(np.float64)
    f4 = cams[:, 12:16].astype(np.float64)
    means = scene["means"].astype(np.float64)
    opac = scene["opacities"].astype(np.float64)
    tot = dict(A_it=0, A_stage=0, A_stage_views=0, VL64_it=0, VL128_it=0, VL_stage=0,
               P2_it=0, P2_stage=0, P2_stage_views=0, sub=0, evals=0, visits_ideal=0,
               A_nosat_it=0, visits_nosat=0, V1_it=0, V1_stage=0, A_union_it=0,
               Ay2_it=0, Ay2_masks=0, Aq4_it=0, Aq4_masks=0, H2_it=0, H2_masks=0, H2_stage=0,
               H2q_it=0, H2q_masks=0, As_it=0, As_masks=0, R_it=0, R_stage=0, R_stage_views=0, P2v_it=0, P2v_stage=0, P2v_stage_views=0, P2v_pairs=0, contrib_visits=0, P2g_it=0, P2g_stage=0, P2g_stage_views=0, P4v_it=0, P4v_stage=0, P4v_stage_views=0)
    for t in tiles:
        tx, ty = t % TX, t // TX
        ls = psi[t]
        ls = ls[ls != 0xFFFF].astype(np.int64)
        ly, rem = ls // 48, ls % 48
        lx, u = rem // 3, rem % 3
        x, y = tx * 16 + lx, ty * 16 + ly
        j = V[y, x, u].astype(np.int64)
        kk = j // s
        for k in range(K):
            sel = np.nonzero(kk == k)[0]
            if sel.size == 0:
                continue
            L = pay[S[t, k]:E[t, k]].astype(np.int64)
            n = L.size
            xs, ys, us, js = x[sel], y[sel], u[sel], j[sel]
            nsub = sel.size
            tot["sub"] += nsub
            if n == 0:
                continue
            A, B, Cc = (rec["conic"][k, L, q].astype(np.float64) for q in range(3))
            col = rec["color"][k, L].astype(np.float64)
            a2, c2 = rec["cov2d"][k, L, 0].astype(np.float64), rec["cov2d"][k, L, 2].astype(np.float64)
            ex = np.sqrt(np.maximum(tau[L] * a2, 0)) * 1.001 + 0.5
            ey = np.sqrt(np.maximum(tau[L] * c2, 0)) * 1.001 + 0.5
            views = np.unique(js)
            mu = {}
            for jj in views:
                p = means[L] @ R[jj].T + tv[jj]
                vis = p[:, 2] >= 0.01
                mx = np.where(vis, f4[jj, 0] * p[:, 0] / p[:, 2] + f4[jj, 2], 1e18)
                my = np.where(vis, f4[jj, 1] * p[:, 1] / p[:, 2] + f4[jj, 3], 1e18)
                mu[jj] = (mx, my)
            # per subpixel: contributing flags, stop index
            stop = np.full(nsub, n, np.int64)  # entries visited: [0, stop) (stop entry included)
            contrib = np.zeros((nsub, n), bool)
            for q in range(nsub):
                mx, my = mu[js[q]]
                dx = mx - (xs[q] + 0.5)
                dy = my - (ys[q] + 0.5)
                pw = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy
                al = np.minimum(0.99, opac[L] * np.exp(np.minimum(pw, 0)))
                ok = (pw <= 0) & (al >= 1 / 255)
                contrib[q] = ok
                T = 1.0
                for e in np.nonzero(ok)[0]:
                    Tn = T * (1 - al[e])
                    if Tn < 1e-4:
                        stop[q] = e + 1
                        break
                    T = Tn
            tot["evals"] += int(stop.sum())

            def boxes(members):
                out = {}
                for jj in np.unique(js[members]):
                    m = members[js[members] == jj]
                    x0, x1, y0, y1 = xs[m].min(), xs[m].max(), ys[m].min(), ys[m].max()
                    bx, by = 0.5 * (x0 + x1) + 0.5, 0.5 * (y0 + y1) + 0.5
                    hx, hy = 0.5 * (x1 - x0), 0.5 * (y1 - y0)
                    mx, my = mu[jj]
                    out[jj] = (np.abs(mx - bx) <= hx + ex) & (np.abs(my - by) <= hy + ey)
                return out

            def boxes_split(members, key):
                out = {}
                for g in np.unique(key[members]):
                    m = members[key[members] == g]
                    x0, x1, y0, y1 = xs[m].min(), xs[m].max(), ys[m].min(), ys[m].max()
                    bx, by = 0.5 * (x0 + x1) + 0.5, 0.5 * (y0 + y1) + 0.5
                    hx, hy = 0.5 * (x1 - x0), 0.5 * (y1 - y0)
                    mx, my = mu[js[m[0]]]
                    out[g] = (np.abs(mx - bx) <= hx + ex) & (np.abs(my - by) <= hy + ey)
                return out

            idx = np.arange(n)
            # ---- A and VL: chunks of 32 consecutive ranks
            for c0 in range(0, nsub, 32):
                mem = np.arange(c0, min(nsub, c0 + 32))
                bx = boxes(mem)
                passm = np.stack([bx[js[q]] & (idx < stop[q]) for q in mem])  # [lanes, n]
                tot["visits_ideal"] += int(passm.sum())
                last = int(stop[mem].max())
                nb = (last + 31) // 32
                tot["A_stage"] += nb
                tot["A_stage_views"] += nb * len(bx)
                for b in range(nb):
                    tot["A_it"] += int(passm[:, b * 32:(b + 1) * 32].sum(1).max())
                lens = np.floor((3 * xs + us + 3 * ys * math.tan(c.slant) - c.center_offset)
                                / c.lens_pitch).astype(np.int64)
                skey = js * 100000 + (lens - lens.min())
                for key, kit, kmk in ((skey, "As_it", "As_masks"),
                                      (js * 2 + (ys % 16 >= 8), "Ay2_it", "Ay2_masks"),
                                      (js * 4 + (ys % 16 >= 8) * 2 + (xs % 16 >= 8), "Aq4_it", "Aq4_masks")):
                    bs = boxes_split(mem, key)
                    pm = np.stack([bs[key[q]] & (idx < stop[q]) for q in mem])
                    tot[kmk] += nb * len(bs)
                    for b in range(nb):
                        tot[kit] += int(pm[:, b * 32:(b + 1) * 32].sum(1).max())
                pn = np.stack([bx[js[q]] for q in mem])
                tot["visits_nosat"] += int(pn.sum())
                for b in range(0, n, 32):
                    tot["A_nosat_it"] += int(pn[:, b:b + 32].sum(1).max())
                um = np.any(passm, 0)
                for b in range(nb):
                    tot["A_union_it"] += int(um[b * 32:(b + 1) * 32].sum())
                for SB, key in ((64, "VL64_it"), (128, "VL128_it")):
                    for b in range(0, last, SB):
                        tot[key] += int(passm[:, b:b + SB].sum(1).max())
            # ---- R: per 32-entry batch, the cluster's not-yet-saturated
            # subpixels repacked (Psi order) into ceil(alive / 32) warps
            last_all = int(stop.max())
            for b in range(0, last_all, 32):
                alive = np.nonzero(stop > b)[0]
                for c0 in range(0, alive.size, 32):
                    mem = alive[c0:c0 + 32]
                    bx = boxes(mem)
                    tot["R_stage"] += 1
                    tot["R_stage_views"] += len(bx)
                    pm = np.stack([bx[js[q]][b:b + 32] & (idx[b:b + 32] < stop[q]) for q in mem])
                    tot["R_it"] += int(pm.sum(1).max())
            # ---- H2: chunks = the top / bottom half of the tile (<= 32 ranks each,
            # overflow split), per-view boxes inside the chunk (and per quadrant)
            half = (ys % 16 >= 8).astype(np.int64)
            for hh in (0, 1):
                memh = np.nonzero(half == hh)[0]
                for c0 in range(0, memh.size, 32):
                    mem = memh[c0:c0 + 32]
                    bx = boxes(mem)
                    last = int(stop[mem].max())
                    nb = (last + 31) // 32
                    tot["H2_stage"] += nb
                    tot["H2_masks"] += nb * len(bx)
                    pm = np.stack([bx[js[q]] & (idx < stop[q]) for q in mem])
                    for b in range(nb):
                        tot["H2_it"] += int(pm[:, b * 32:(b + 1) * 32].sum(1).max())
                    key = js * 2 + (xs % 16 >= 8)
                    bs = boxes_split(mem, key)
                    tot["H2q_masks"] += nb * len(bs)
                    pm = np.stack([bs[key[q]] & (idx < stop[q]) for q in mem])
                    for b in range(nb):
                        tot["H2q_it"] += int(pm[:, b * 32:(b + 1) * 32].sum(1).max())
            # ---- V1: one chunk per view (lanes = that view's subpixels)
            for jj in np.unique(js):
                mem = np.nonzero(js == jj)[0]
                bx = boxes(mem)
                passm = np.stack([bx[jj] & (idx < stop[q]) for q in mem])
                last = int(stop[mem].max())
                nb = (last + 31) // 32
                tot["V1_stage"] += nb
                for b in range(nb):
                    tot["V1_it"] += int(passm[:, b * 32:(b + 1) * 32].sum(1).max())
            # ---- P2: chunks of up to 64 ranks, lanes hold ranks (2l, 2l+1)
            nch = max(1, math.ceil(nsub / 64))
            bounds = np.linspace(0, nsub, nch + 1).round().astype(int)
            for ci in range(nch):
                mem = np.arange(bounds[ci], bounds[ci + 1])
                bx = boxes(mem)
                lanes = [mem[q:q + 2] for q in range(0, mem.size, 2)]
                last = int(stop[mem].max())
                nb = (last + 31) // 32
                tot["P2_stage"] += nb
                tot["P2_stage_views"] += nb * len(bx)
                lm = np.stack([np.any(np.stack([bx[js[q]] & (idx < stop[q]) for q in ln]), 0)
                               for ln in lanes])
                for b in range(nb):
                    tot["P2_it"] += int(lm[:, b * 32:(b + 1) * 32].sum(1).max())

            # ---- P2v: same-view pairs (each view run padded to an even length),
            # chunks of <= 32 pairs inside the cluster segment
            pairs = []
            for jj in np.unique(js):
                m = np.nonzero(js == jj)[0]
                for q in range(0, m.size, 2):
                    pairs.append(m[q:q + 2])
            tot["P2v_pairs"] += len(pairs)
            for c0 in range(0, len(pairs), 32):
                lanes = pairs[c0:c0 + 32]
                mem = np.concatenate(lanes)
                bx = boxes(mem)
                last = int(stop[mem].max())
                nb = (last + 31) // 32
                tot["P2v_stage"] += nb
                tot["P2v_stage_views"] += nb * len(bx)
                lm = np.stack([bx[js[ln[0]]] & (idx < stop[ln].max()) for ln in lanes])
                for b in range(nb):
                    tot["P2v_it"] += int(lm[:, b * 32:(b + 1) * 32].sum(1).max())
            for q in range(nsub):
                tot["contrib_visits"] += int((contrib[q] & (idx < stop[q])).sum())
            # ---- P2g: P2v lanes, chunks of 32 lanes then the remainder (greedy);
            # P4v: four same-view subpixels per lane (view runs padded to 4)
            for key, per in (("P2g", 2), ("P4v", 4)):
                groups = []
                for jj in np.unique(js):
                    m = np.nonzero(js == jj)[0]
                    for q in range(0, m.size, per):
                        groups.append(m[q:q + per])
                for c0 in range(0, len(groups), 32):
                    lanes = groups[c0:c0 + 32]
                    mem = np.concatenate(lanes)
                    bx = boxes(mem)
                    last = int(stop[mem].max())
                    nb = (last + 31) // 32
                    tot[key + "_stage"] += nb
                    tot[key + "_stage_views"] += nb * len(bx)
                    lm = np.stack([bx[js[ln[0]]] & (idx < stop[ln].max()) for ln in lanes])
                    for b in range(nb):
                        tot[key + "_it"] += int(lm[:, b * 32:(b + 1) * 32].sum(1).max())
    print(name, "tiles", len(tiles), tot)
    A = tot["A_it"]
    print(f"visits(ideal lane work)/32 = {tot['visits_ideal']/32:.0f}  A iterations {A}  "
          f"util {tot['visits_ideal']/32/A:.3f}")
    print(f"no saturation: ideal {tot['visits_nosat']/32:.0f} A {tot['A_nosat_it']} "
          f"util {tot['visits_nosat']/32/tot['A_nosat_it']:.3f}")
    print(f"masks: A {tot['A_stage_views']} y2 {tot['Ay2_masks']} q4 {tot['Aq4_masks']} stripe {tot['As_masks']}")
    print(f"H2 masks {tot['H2_masks']} stage {tot['H2_stage']}  H2q masks {tot['H2q_masks']}")
    print(f"repack: stage batches {tot['R_stage']} (views {tot['R_stage_views']}) vs A {tot['A_stage']} (views {tot['A_stage_views']})")
    for k in ("R_it", "VL64_it", "VL128_it", "P2_it", "V1_it", "A_union_it", "Ay2_it", "Aq4_it", "H2_it", "H2q_it", "As_it"):
        print(f"{k}: {tot[k]} ({tot[k]/A:.3f} of A)")
    print(f"stage batches A {tot['A_stage']} (views {tot['A_stage_views']}), P2 {tot['P2_stage']} "
          f"(views {tot['P2_stage_views']})")


if __name__ == "__main__":
    main()

