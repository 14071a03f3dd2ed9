"""ctypes binding of libcoherent_raster.so (include/coherent_raster.h).

Argument marshalling only: every step of the rendering path runs in the
library's CUDA kernels.  There is no CPU fallback: if the shared library is
missing this module raises at import of the renderer.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

STATUS = {
    0: "CR_OK", 1: "CR_ERR_INVALID_ARG", 2: "CR_ERR_INVALID_CONFIG", 3: "CR_ERR_CONFIG_MISMATCH",
    4: "CR_ERR_TILE_ID_OVERFLOW", 5: "CR_ERR_NONFINITE", 6: "CR_ERR_NOT_READY",
    7: "CR_ERR_OUT_OF_MEMORY", 8: "CR_ERR_CUDA", 9: "CR_ERR_CAPACITY",
}

# exported symbols, in header order (tests check the library exports all of them)
SYMBOLS = [
    "cr_create", "cr_destroy", "cr_set_stream", "cr_synchronize", "cr_last_error", "cr_status_string", "cr_version",
    "cr_upload_gaussians", "cr_set_display", "cr_set_camera_rig", "cr_make_orbit_rig",
    "cr_render_interlaced", "cr_get_view_map", "cr_get_remap", "cr_get_sorted_pairs",
    "cr_get_ranges", "cr_get_depths", "cr_get_counts",
]


class CrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Display(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("num_views", C.c_int32),
                ("lens_pitch", C.c_double), ("slant", C.c_double), ("center_offset", C.c_double),
                ("view_cone", C.c_double), ("tile_size", C.c_int32)]


class Camera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float)]


class RenderOpts(C.Structure):
    _fields_ = [("cluster_size", C.c_int32), ("remap", C.c_int32), ("kernel", C.c_int32),
                ("background", C.c_float * 3), ("output_format", C.c_int32),
                ("tile_row_begin", C.c_int32), ("tile_row_end", C.c_int32),
                ("flags", C.c_int32), ("view_batch", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("visible_ik", C.c_int64), ("culled_near", C.c_int64),
                ("culled_degenerate", C.c_int64), ("culled_opacity", C.c_int64),
                ("num_clusters", C.c_int32), ("bit_k", C.c_int32), ("launches", C.c_int32),
                ("emit_fallback", C.c_int32), ("ms_preprocess", C.c_float), ("ms_bin", C.c_float),
                ("ms_sort", C.c_float), ("ms_composite", C.c_float), ("ms_total", C.c_float),
                ("device_bytes", C.c_int64), ("evals", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load(path: str | None = None):
    """Load the shared library (raises if it was not built).  CR_LIB overrides
    the path (A/B timing of alternative builds)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("CR_LIB") or LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2605_04509_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, st = C.c_void_p, C.c_int
    sz = C.POINTER(C.c_size_t)

    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)

    sig("cr_create", st, C.c_int, vp, C.POINTER(vp))
    sig("cr_destroy", None, vp)
    sig("cr_set_stream", st, vp, vp)
    sig("cr_synchronize", st, vp)
    sig("cr_last_error", C.c_char_p, vp)
    sig("cr_status_string", C.c_char_p, st)
    sig("cr_version", C.c_char_p)
    sig("cr_upload_gaussians", st, vp, C.c_int64, C.c_int, vp, vp, vp, vp, vp, C.c_int)
    sig("cr_set_display", st, vp, C.POINTER(Display))
    sig("cr_set_camera_rig", st, vp, C.c_int32, vp, C.c_float)
    sig("cr_make_orbit_rig", st, C.POINTER(Display), C.POINTER(C.c_float * 3),
        C.POINTER(C.c_float * 3), C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, vp)
    sig("cr_render_interlaced", st, vp, C.POINTER(RenderOpts), vp, C.c_size_t, C.c_int,
        C.POINTER(Stats))
    sig("cr_get_view_map", st, vp, vp, sz)
    sig("cr_get_remap", st, vp, vp, sz)
    sig("cr_get_sorted_pairs", st, vp, vp, vp, sz)
    sig("cr_get_ranges", st, vp, vp, vp, sz)
    sig("cr_get_depths", st, vp, vp, sz)
    sig("cr_get_counts", st, vp, vp, sz)
    _lib = L
    return L


def check(L, ctx, status: int):
    if status != 0:
        msg = L.cr_last_error(ctx) if ctx else b""
        raise CrError(status, (msg or b"").decode(errors="replace"))
