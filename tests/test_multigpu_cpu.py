"""Host logic of the row-band split and the band gather, on CPU with the
gloo backend at world size 2 (the NCCL path uses the same code on B200)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_04509_b200 import multigpu as mg


def test_band_rows_partition():
    for TY in (1, 9, 135, 270):
        for world in (1, 2, 3, 4, 8):
            if world > TY:
                continue
            bands = [mg.band_rows(TY, world, r) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == TY
            assert all(bands[q][1] == bands[q + 1][0] for q in range(world - 1))
            sizes = [b - a for a, b in bands]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_balanced_bands():
    rng = np.random.default_rng(0)
    for TY in (9, 135, 270):
        w = rng.gamma(0.5, 1.0, TY) * (np.arange(TY) > TY // 3)  # skewed, with empty rows
        for world in (1, 2, 3, 8):
            bands = mg.balanced_bands(w, world)
            assert bands[0][0] == 0 and bands[-1][1] == TY
            assert all(b[1] > b[0] for b in bands)
            assert all(bands[q][1] == bands[q + 1][0] for q in range(world - 1))
            loads = [w[a:b].sum() for a, b in bands]
            # no band exceeds the ideal share by more than its heaviest single row
            assert max(loads) <= w.sum() / world + w.max() + 1e-6
    assert mg.balanced_bands(np.ones(8), 8) == [(q, q + 1) for q in range(8)]


def test_refine_bands_converges_to_true_cost():
    # the model (uniform pairs) mispredicts a true per-row cost; refining with
    # measured band costs must approach the true balanced split
    TY, world = 135, 8
    rng = np.random.default_rng(1)
    true = 1.0 + 4.0 * np.exp(-((np.arange(TY) - 60) / 12.0) ** 2) + rng.uniform(0, 0.2, TY)
    model = np.ones(TY)
    bands = mg.balanced_bands(model, world)
    worst0 = max(true[a:b].sum() for a, b in bands)
    w = model
    for _ in range(4):
        costs = [true[a:b].sum() for a, b in bands]
        bands, w = mg.refine_bands(w, bands, costs, world)
        assert bands[0][0] == 0 and bands[-1][1] == TY
        assert all(bands[q][1] == bands[q + 1][0] and bands[q][1] > bands[q][0] for q in range(world - 1))
    worst = max(true[a:b].sum() for a, b in bands)
    ideal = true.sum() / world
    assert worst < worst0
    assert worst <= ideal + 2 * true.max()
    # exact model: refinement keeps the balanced split
    b0 = mg.balanced_bands(true, world)
    b1, _ = mg.refine_bands(true, b0, [true[a:b].sum() for a, b in b0], world)
    assert b1 == b0


def test_pose_split_covers_all():
    got = sorted(sum((mg.pose_split(256, 8, r) for r in range(8)), []))
    assert got == list(range(256)) and len(mg.pose_split(256, 8, 3)) == 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame_ref(H, W):
    # deterministic stand-in for a rendered frame: value depends on (y, x, u)
    y, x, u = np.meshgrid(np.arange(H), np.arange(W), np.arange(3), indexing="ij")
    return ((y * 7 + x * 3 + u * 11) % 251).astype(np.uint8)


def _worker(rank, world, port, H, W, q, balanced=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    TY = (H + 15) // 16
    bands = mg.balanced_bands(np.linspace(0, 1, TY) ** 3, world) if balanced else None
    bg = mg.BandGather(H, W, TY, world, rank, "cpu", bands=bands)
    ref = _frame_ref(H, W)
    y0, y1 = mg.band_pixel_rows(H, TY, world, rank, bands)
    bg.out.copy_(torch.from_numpy(ref[y0:y1]))  # "render" this rank's band
    bg.gather()
    full = bg.frame().numpy()
    # unpadded: each rank receives exactly the other ranks' rows
    q.put((rank, bool(np.array_equal(full, ref)) and bg.bytes_received() == (H - (y1 - y0)) * W * 3,
           bg.rows))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H,balanced", [(144, False), (138, False), (2160, False), (2160, True)])
def test_gloo_world2_band_gather(H, balanced):
    W, world = 40, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, q, balanced))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _ in res)
    assert res[0][2][1] == res[1][2][0]  # contiguous bands
