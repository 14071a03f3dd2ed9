"""Row-band sharding of the interlaced frame over the GPUs of one node
(SURVEY §8(e)).  Gaussians are replicated; rank r renders tile rows
band_rows(TY, R, r) of the frame (keys keep global tile ids, so its pairs are
the full frame's pairs filtered to the band); every rank renders straight into
its rows of a full-frame buffer and the bands are exchanged in place with one
broadcast per band (NCCL over NVLink on B200, gloo in the CPU tests) — no
padding to the tallest band.  Pose batches (config E) split the
poses round-robin with no collective.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def band_rows(TY: int, world: int, rank: int):
    """Contiguous tile-row band [r0, r1) of `rank`; sizes differ by <= 1 row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(TY, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def balanced_bands(weights, world: int):
    """Contiguous tile-row bands of ~equal total weight (weights[ty] = cost of
    tile row ty, e.g. its Gaussian-tile pairs from a calibration frame);
    every band gets >= 1 row.  Returns [(r0, r1)] * world."""
    import numpy as np
    w = np.asarray(weights, np.float64)
    TY = w.shape[0]
    if world > TY:
        raise ValueError("more ranks than tile rows")
    cum = np.concatenate([[0.0], np.cumsum(np.maximum(w, 0) + 1e-9)])
    cuts = [0]
    for q in range(1, world):
        target = cum[-1] * q / world
        c = int(np.searchsorted(cum, target))
        c = max(c, cuts[-1] + 1)           # at least one row per band
        c = min(c, TY - (world - q))       # leave a row for each later band
        cuts.append(c)
    cuts.append(TY)
    return [(cuts[q], cuts[q + 1]) for q in range(world)]


def refine_bands(weights, bands, costs, world: int):
    """One refinement step of the band split from MEASURED per-band costs.

    weights[ty]: the current per-row cost model (e.g. calibration pair counts);
    bands: the split that was measured; costs[b]: band b's measured variable
    time (total minus the replicated per-rank part).  Every row of band b is
    rescaled by costs[b] / sum(weights in b), which keeps the within-band shape
    of the model and corrects its scale where it mispredicts (e.g. rows of
    background splats that are cheap to bin but slow to composite); the new
    split balances the corrected weights.  Returns (new_bands, new_weights)."""
    import numpy as np
    w = np.asarray(weights, np.float64).copy()
    for (r0, r1), c in zip(bands, costs):
        tot = w[r0:r1].sum()
        if tot > 0:
            w[r0:r1] *= max(float(c), 0.0) / tot
        else:
            w[r0:r1] = max(float(c), 0.0) / max(1, r1 - r0)
    return balanced_bands(w, world), w


def _pix(H, r0, r1):
    return r0 * 16, min(H, r1 * 16)


def band_pixel_rows(H: int, TY: int, world: int, rank: int, bands=None):
    r0, r1 = bands[rank] if bands else band_rows(TY, world, rank)
    return _pix(H, r0, r1)


class BandGather:
    """Full-frame buffer of one rank; the rank renders its band straight into
    its rows (row-major, so the band is a contiguous slice) and gather()
    fills the other ranks' rows in place with one broadcast per band (NCCL
    over NVLink): every rank receives exactly the frame's other rows — no
    padding to the tallest band (balanced bands differ in height)."""

    def __init__(self, H: int, W: int, TY: int, world: int, rank: int, device, dtype=torch.uint8,
                 bands=None):
        self.H, self.W, self.TY, self.world, self.rank = H, W, TY, world, rank
        self.bands = bands
        self.rows = bands[rank] if bands else band_rows(TY, world, rank)
        self.full = torch.zeros((H, W, 3), dtype=dtype, device=device)
        self.pix = [band_pixel_rows(H, TY, world, q, bands) for q in range(world)]
        y0, y1 = self.pix[rank]
        self.out = self.full[y0:y1]  # what the renderer writes (contiguous rows)

    def gather(self, group=None) -> torch.Tensor:
        """Fill every other rank's band rows; returns the full frame."""
        if self.world == 1:
            return self.full
        on_host = dist.get_backend(group) != "nccl" and self.full.device.type != "cpu"
        buf = self.full.cpu() if on_host else self.full  # gloo with CUDA tensors (tests)
        for q, (y0, y1) in enumerate(self.pix):
            if y1 > y0:
                dist.broadcast(buf[y0:y1], src=q, group=group)
        if on_host:
            self.full.copy_(buf)
        return self.full

    def frame(self) -> torch.Tensor:
        return self.full

    def bytes_received(self) -> int:
        y0, y1 = self.pix[self.rank]
        return (self.H - (y1 - y0)) * self.W * 3 * self.full.element_size()


def row_pair_weights(renderer, cluster_size: int):
    """Per-tile-row Gaussian-tile pair counts of the last full-frame render
    (cr_get_ranges): the load-balancing weights for balanced_bands."""
    import numpy as np
    K = -(-renderer.display["num_views"] // cluster_size)
    S, E = renderer.ranges(K)
    per_tile = (E.astype(np.int64) - S.astype(np.int64)).sum(axis=1)
    return per_tile.reshape(renderer.TY, renderer.TX).sum(axis=1)


def pose_split(n_poses: int, world: int, rank: int):
    """Round-robin pose indices of `rank` (config E)."""
    return list(range(rank, n_poses, world))
