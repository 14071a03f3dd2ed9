"""Python face of the C ABI: `CoherentRaster` (one context per GPU).

Thin marshalling over libcoherent_raster.so: PyTorch supplies device memory
(output tensors) and the CUDA stream; every stage of the path runs in the
library's kernels.  Names follow the paper: cluster_size = |V_k|,
remap = View-coherent Remapping, view map V (Eqs.1-3).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N


def _ptr(x):
    if isinstance(x, torch.Tensor):
        return x.data_ptr()
    return x.ctypes.data


def _as_f32(x, device):
    """Contiguous float32 tensor on `device` (device) or numpy (host)."""
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=device, dtype=torch.float32).contiguous()
    return np.ascontiguousarray(x, dtype=np.float32)


class CoherentRaster:
    """Subpixel-level light-field 3DGS rasterizer on one CUDA device."""

    def __init__(self, device: int | str | torch.device = 0, stream: torch.cuda.Stream | None = None):
        self._L = N.load()
        dev = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
        if dev.type != "cuda":
            raise ValueError("CoherentRaster runs on CUDA devices only (no CPU fallback)")
        self.device = torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())
        self._stream = stream or torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        N.check(self._L, None, self._L.cr_create(self.device.index, C.c_void_p(self._stream.cuda_stream),
                                                 C.byref(ctx)))
        self._ctx = ctx
        self.display = None
        self.M = 0
        self.last_stats = None
        self._keep = []

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_ctx", None):
            self._L.cr_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, status):
        N.check(self._L, self._ctx, status)

    @property
    def stream(self):
        return self._stream

    def set_stream(self, stream: torch.cuda.Stream):
        self._stream = stream
        self._check(self._L.cr_set_stream(self._ctx, C.c_void_p(stream.cuda_stream)))

    def synchronize(self):
        """Wait for every rendered frame, including async_out host copies."""
        self._check(self._L.cr_synchronize(self._ctx))

    @staticmethod
    def version() -> str:
        return N.load().cr_version().decode()

    # ------------------------------------------------------------------ inputs
    def upload_gaussians(self, scene: dict, on_device: bool | None = None):
        """D1: means [M,3], quats [M,4] (w,x,y,z), scales [M,3],
        opacities [M], sh [M,(d+1)^2,3]; numpy (host) or CUDA tensors."""
        M = int(scene["means"].shape[0])
        deg = int(scene["sh_degree"])
        keys = ("means", "quats", "scales", "opacities", "sh")
        dev = on_device if on_device is not None else isinstance(scene["means"], torch.Tensor)
        arrs = [_as_f32(scene[k], self.device) if dev else np.ascontiguousarray(
            scene[k].cpu().numpy() if isinstance(scene[k], torch.Tensor) else scene[k], np.float32)
            for k in keys]
        ptrs = [C.c_void_p(_ptr(a)) if M else None for a in arrs]
        self._check(self._L.cr_upload_gaussians(self._ctx, M, deg, *ptrs, int(bool(dev))))
        self.M = M

    def set_display(self, width, height, num_views, lens_pitch, slant, center_offset,
                    view_cone=53.0):
        """§3.1 display: builds V (Eqs.1-3) and Psi on the device."""
        d = N.Display(int(width), int(height), int(num_views), float(lens_pitch), float(slant),
                      float(center_offset), float(view_cone), 16)
        self._check(self._L.cr_set_display(self._ctx, C.byref(d)))
        self.display = dict(width=int(width), height=int(height), num_views=int(num_views),
                            lens_pitch=float(lens_pitch), slant=float(slant),
                            center_offset=float(center_offset), view_cone=float(view_cone))
        self.TX, self.TY = (int(width) + 15) // 16, (int(height) + 15) // 16

    def set_camera_rig(self, cams, znear: float = 0.01):
        """Target views v_j: [N,16] float32 rows (R[9], t[3], fx, fy, cx, cy)."""
        a = np.ascontiguousarray(cams.cpu().numpy() if isinstance(cams, torch.Tensor) else cams,
                                 np.float32).reshape(-1, 16)
        self._check(self._L.cr_set_camera_rig(self._ctx, a.shape[0], C.c_void_p(a.ctypes.data),
                                              float(znear)))

    @staticmethod
    def make_orbit_rig(display: dict, look_at=(0, 0, 0), up=(0, 1, 0), radius=4.0, height=0.8,
                       yaw_deg=0.0, pitch_deg=0.0, fov_y_deg=40.0) -> np.ndarray:
        L = N.load()
        d = N.Display(display["width"], display["height"], display["num_views"],
                      display["lens_pitch"], display["slant"], display["center_offset"],
                      display.get("view_cone", 53.0), 16)
        out = np.zeros((display["num_views"], 16), np.float32)
        la = (C.c_float * 3)(*look_at)
        upv = (C.c_float * 3)(*up)
        N.check(L, None, L.cr_make_orbit_rig(C.byref(d), C.byref(la), C.byref(upv), radius, height,
                                             yaw_deg, pitch_deg, fov_y_deg,
                                             C.c_void_p(out.ctypes.data)))
        return out

    # ------------------------------------------------------------------ render
    def band_shape(self, rows=None):
        W, H = self.display["width"], self.display["height"]
        r0, r1 = rows if rows else (0, self.TY)
        y0, y1 = r0 * 16, min(H, r1 * 16)
        return (max(0, y1 - y0), W, 3)

    def render(self, cluster_size: int = 8, remap: bool = True, kernel: int | None = None,
               background=(0.0, 0.0, 0.0), output_format: str = "rgb8", rows=None, out=None,
               stats: bool = False, count_evals: bool = False, fullframe: bool = False,
               view_frames: bool = False, view_batch: int = 0, async_out: bool = False):
        """One interlaced frame I_LF (Alg.1) for tile rows `rows`
        (None = full frame).  Returns a CUDA tensor [rows*16, W, 3] (uint8 or
        float32); `out` may be a preallocated CUDA tensor or a host tensor /
        numpy array (copied back inside the call).  fullframe=True renders
        every view full frame at cluster size s, then interlaces (s=1: the
        traditional baseline).  view_frames=True returns those per-view frames
        [N, rows*16, W, 3] instead (the per-view images of P:478).
        view_batch=B renders the full-frame baseline B views per pass (the
        paper's "3DGS (batch=B)"; 1 = plain per-view 3DGS).
        async_out=True with a host `out` (pinned): the copy back overlaps the
        next frame; `out` is valid after synchronize()."""
        if kernel is None:
            kernel = 0 if remap else 1
        fmt = 0 if output_format == "rgb8" else 1
        r0, r1 = rows if rows else (0, 0)
        opts = N.RenderOpts(int(cluster_size), int(bool(remap)), int(kernel),
                            (C.c_float * 3)(*[float(b) for b in background]), fmt, int(r0), int(r1),
                            (1 if count_evals else 0) | (2 if fullframe else 0)
                            | (4 if view_frames else 0) | (8 if async_out else 0), int(view_batch))
        dtype = torch.uint8 if fmt == 0 else torch.float32
        if self.display is None:  # let the library report CR_ERR_NOT_READY
            out = torch.empty(1, dtype=dtype, device=self.device) if out is None else out
        shape = self.band_shape(rows) if self.display is not None else (1,)
        if view_frames and self.display is not None:
            shape = (self.display["num_views"],) + tuple(shape)
        if out is None:
            out = torch.empty(shape, dtype=dtype, device=self.device)
        on_dev = isinstance(out, torch.Tensor) and out.is_cuda
        if isinstance(out, torch.Tensor):
            assert out.is_contiguous() and out.dtype == dtype
            nbytes = out.numel() * out.element_size()
        else:
            assert out.flags.c_contiguous and out.dtype == (np.uint8 if fmt == 0 else np.float32)
            nbytes = out.nbytes
        st = N.Stats() if (stats or count_evals) else None
        self._check(self._L.cr_render_interlaced(self._ctx, C.byref(opts), C.c_void_p(_ptr(out)),
                                                 nbytes, int(on_dev),
                                                 C.byref(st) if st is not None else None))
        self.last_stats = st.as_dict() if st is not None else None
        return out

    # ------------------------------------------------------------------ introspection
    def _get(self, fn, dtype, *extra_nulls):
        n = C.c_size_t(0)
        self._check(fn(self._ctx, *([None] * (1 + len(extra_nulls))), C.byref(n)))
        arrs = [np.zeros(n.value, dtype) for _ in range(1 + len(extra_nulls))]
        self._check(fn(self._ctx, *[C.c_void_p(a.ctypes.data) for a in arrs], C.byref(n)))
        return arrs if extra_nulls else arrs[0]

    def view_map(self) -> np.ndarray:
        d = self.display
        return self._get(self._L.cr_get_view_map, np.uint8).reshape(d["height"], d["width"], 3)

    def remap_table(self) -> np.ndarray:
        return self._get(self._L.cr_get_remap, np.uint16).reshape(self.TY * self.TX, 768)

    def sorted_pairs(self):
        n = C.c_size_t(0)
        self._check(self._L.cr_get_sorted_pairs(self._ctx, None, None, C.byref(n)))
        k = np.zeros(n.value, np.uint64)
        p = np.zeros(n.value, np.uint32)
        self._check(self._L.cr_get_sorted_pairs(self._ctx, C.c_void_p(k.ctypes.data),
                                                C.c_void_p(p.ctypes.data), C.byref(n)))
        return k, p

    def ranges(self, K):
        S, E = self._get(self._L.cr_get_ranges, np.uint32, None)
        return S.reshape(-1, K), E.reshape(-1, K)

    def depths(self, K):
        return self._get(self._L.cr_get_depths, np.float32).reshape(K, self.M)

    def counts(self, K):
        return self._get(self._L.cr_get_counts, np.uint32).reshape(K, self.M)
