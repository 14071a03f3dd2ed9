"""B200-native subpixel light-field 3DGS rasterizer (CoherentRaster, arXiv 2605.04509).

Public API: :class:`CoherentRaster` (C ABI in include/coherent_raster.h,
kernels in csrc/), seeded inputs in :mod:`synthetic`, row-band sharding over
NCCL in :mod:`multigpu`.
"""
from .synthetic import CONFIGS  # noqa: F401

__all__ = ["CoherentRaster", "CONFIGS"]


def __getattr__(name):
    if name == "CoherentRaster":
        from .raster import CoherentRaster
        return CoherentRaster
    raise AttributeError(name)
