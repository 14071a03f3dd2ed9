"""Row-band sharding of the interlaced frame over the GPUs of one node
(SURVEY §8(e)).  Gaussians are replicated; rank r renders tile rows
band_rows(TY, R, r) of the frame (keys keep global tile ids, so its pairs are
the full frame's pairs filtered to the band); the RGB8 bands are padded to a
common height and assembled with one all_gather_into_tensor (NCCL over
NVLink on B200, gloo in the CPU tests).  Pose batches (config E) split the
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


def band_pixel_rows(H: int, TY: int, world: int, rank: int):
    r0, r1 = band_rows(TY, world, rank)
    return r0 * 16, min(H, r1 * 16)


def padded_band_height(H: int, TY: int, world: int) -> int:
    return max(band_pixel_rows(H, TY, world, q)[1] - band_pixel_rows(H, TY, world, q)[0]
               for q in range(world))


def assemble(gathered: torch.Tensor, H: int, TY: int, world: int) -> torch.Tensor:
    """Full frame [H, W, 3] from the all-gathered padded bands [world*hp, W, 3]."""
    hp = gathered.shape[0] // world
    parts = []
    for q in range(world):
        y0, y1 = band_pixel_rows(H, TY, world, q)
        parts.append(gathered[q * hp:q * hp + (y1 - y0)])
    return torch.cat(parts, 0)


class BandGather:
    """Preallocated padded band buffer + gather target for one rank."""

    def __init__(self, H: int, W: int, TY: int, world: int, rank: int, device, dtype=torch.uint8):
        self.H, self.W, self.TY, self.world, self.rank = H, W, TY, world, rank
        self.rows = band_rows(TY, world, rank)
        y0, y1 = band_pixel_rows(H, TY, world, rank)
        self.hp = padded_band_height(H, TY, world)
        self.band = torch.zeros((self.hp, W, 3), dtype=dtype, device=device)
        self.out = self.band[:y1 - y0]  # what the renderer writes
        self.full = (torch.empty((world * self.hp, W, 3), dtype=dtype, device=device)
                     if world > 1 else None)

    def gather(self, group=None) -> torch.Tensor:
        """All-gather the padded bands; returns the padded stack (or the band at world 1)."""
        if self.world == 1:
            return self.band
        dist.all_gather_into_tensor(self.full, self.band, group=group)
        return self.full

    def frame(self) -> torch.Tensor:
        if self.world == 1:
            return self.out
        return assemble(self.full, self.H, self.TY, self.world)


def pose_split(n_poses: int, world: int, rank: int):
    """Round-robin pose indices of `rank` (config E)."""
    return list(range(rank, n_poses, world))
