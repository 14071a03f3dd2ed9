"""CPU oracle for the CoherentRaster subpixel light-field rasterizer.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2605_04509_b200``) never imports it; the
two share no code (see DESIGN.md §3 and oracle/oracle.cpp's header).

The arithmetic lives in ``oracle.cpp`` (plain C++17, ``-O2 -ffp-contract=off``,
no fast-math).  This module only compiles it (gcc) and marshals numpy arrays
through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
# Mutation testing only (tools/oracle_mutations.py): build a planted-mutation
# copy of oracle.cpp instead, into its own library next to it.
if os.environ.get("CR_ORACLE_MUTANT_SRC"):
    _SRC = os.environ["CR_ORACLE_MUTANT_SRC"]
    _LIB = os.path.splitext(_SRC)[0] + ".so"
_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-fPIC", "-shared",
          "-pthread"]
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (gcc); returns the path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["g++", *_FLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = _bind(C.CDLL(build()))
    return _lib


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def _bind(L):
    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)

    vp = C.c_void_p
    sig("cro_view_index", C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
        C.c_double)
    sig("cro_gaussian_constants", None, C.c_int64, _f32p, _f32p, _f32p, _f32p, _f32p)
    sig("cro_project_mean", C.c_int, _f32p, _f32p, C.c_float, _f32p, _f32p)
    sig("cro_cov2d", C.c_int, _f32p, C.c_int, C.c_int, _f32p, _f32p, _f32p)
    sig("cro_tileset", C.c_int64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float,
        C.c_float, C.c_float, C.c_int, C.c_int, _i32p, C.c_int64)
    sig("cro_sh_basis", None, C.c_int, _f64p, _f64p)
    sig("cro_eval_sh", None, C.c_int, _f32p, _f64p, _f64p)
    sig("cro_blend", C.c_float, _f32p, C.c_int, C.c_float, C.c_float, C.c_float)
    sig("cro_create", vp, C.c_int)
    sig("cro_destroy", None, vp)
    sig("cro_threads", C.c_int, vp)
    sig("cro_set_tile_pad", None, vp, C.c_float)
    sig("cro_set_scene", C.c_int, vp, C.c_int64, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p)
    sig("cro_get_constants", None, vp, _f32p, _f32p)
    sig("cro_set_display_tan", C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
        C.c_double)
    sig("cro_set_display", C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
        C.c_double)
    sig("cro_get_view_map", None, vp, _u8p)
    sig("cro_get_remap", None, vp, C.c_int, _u16p)
    sig("cro_set_rig", C.c_int, vp, C.c_int, _f32p, C.c_float)
    sig("cro_clusters", C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
        C.POINTER(C.c_int))
    sig("cro_render", C.c_int, vp, C.c_int, C.c_int, C.c_int, _f32p, vp, C.c_int64, C.c_int)
    sig("cro_num_clusters", C.c_int, vp)
    sig("cro_bit_k", C.c_int, vp)
    sig("cro_num_pairs", C.c_int64, vp)
    sig("cro_num_evals", C.c_int64, vp)
    sig("cro_get_pairs", None, vp, _u64p, _u32p)
    sig("cro_get_ranges", None, vp, _u32p, _u32p)
    sig("cro_get_image", None, vp, _f32p)
    sig("cro_get_records", None, vp, vp, vp, vp, vp, vp, vp)
    sig("cro_render_bruteforce", C.c_int, vp, _f32p)
    sig("cro_render_views", C.c_int, vp, _f32p)
    return L


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- unit calls
def view_index(x, y, u, N, Lx, tan_alpha, Koff) -> int:
    """O1: Eqs.1-3 for one subpixel."""
    return lib().cro_view_index(x, y, u, N, Lx, tan_alpha, Koff)


def gaussian_constants(quats, scales, opac):
    """O4: Sigma3D (6 floats, 00 01 02 11 12 22) and tau = 2 ln(255 o)."""
    q, s, o = _f32(quats).reshape(-1, 4), _f32(scales).reshape(-1, 3), _f32(opac).reshape(-1)
    M = o.shape[0]
    cov = np.zeros((M, 6), np.float32)
    tau = np.zeros(M, np.float32)
    lib().cro_gaussian_constants(M, q, s, o, cov, tau)
    return cov, tau


def cam16(cam) -> np.ndarray:
    """Camera dict/array -> 16 floats (R[9] row-major world->camera, t[3], fx, fy, cx, cy)."""
    if isinstance(cam, dict):
        return _f32(np.concatenate([np.asarray(cam["R"], np.float32).reshape(9),
                                    np.asarray(cam["t"], np.float32).reshape(3),
                                    np.asarray([cam["fx"], cam["fy"], cam["cx"], cam["cy"]],
                                               np.float32)]))
    return _f32(cam).reshape(16)


def project_mean(cam, mu, znear=0.01):
    """O5 / Eq.5: (mu2d, depth, visible)."""
    out = np.zeros(2, np.float32)
    d = np.zeros(1, np.float32)
    vis = lib().cro_project_mean(cam16(cam), _f32(mu).reshape(3), znear, out, d)
    return out, float(d[0]), bool(vis)


def cov2d(cam, W, H, mu, cov6):
    """O6: (a, b, c, det) after +0.3 dilation and the non-degenerate flag."""
    out = np.zeros(4, np.float32)
    ok = lib().cro_cov2d(cam16(cam), W, H, _f32(mu).reshape(3), _f32(cov6).reshape(6), out)
    return out, bool(ok)


def tileset(m, abcd, tau, TX, TY):
    """O7 AccuTile reading: sorted tile ids of one view's ellipse."""
    cap = 1 << 16
    buf = np.zeros(cap, np.int32)
    a, b, c, det = [float(v) for v in abcd]
    n = lib().cro_tileset(float(m[0]), float(m[1]), a, b, c, det, float(tau), TX, TY, buf, cap)
    if n < 0:
        raise ValueError("tile set too large")
    return buf[:n].copy()


def sh_basis(deg, d):
    out = np.zeros(16, np.float64)
    lib().cro_sh_basis(deg, np.ascontiguousarray(d, np.float64), out)
    return out


def eval_sh(deg, sh, d):
    """O11: unclamped SH colour + 0.5 (3DGS convention)."""
    out = np.zeros(3, np.float64)
    lib().cro_eval_sh(deg, _f32(sh).reshape(-1), np.ascontiguousarray(d, np.float64), out)
    return out


def blend(splats, px, py, bg=0.0) -> float:
    """O12 for one subpixel; splats rows (mx, my, A, B, C, o, colour) front to back."""
    s = _f32(splats).reshape(-1, 7)
    return float(lib().cro_blend(np.ascontiguousarray(s.reshape(-1)), s.shape[0], px, py, bg))


def clusters(N, s):
    """O3: (K, Bit_K, representatives)."""
    K = C.c_int()
    b = C.c_int()
    L = lib()
    if L.cro_clusters(N, s, C.byref(K), C.byref(b), None) != 0:
        raise ValueError("bad clustering")
    rep = (C.c_int * K.value)()
    L.cro_clusters(N, s, C.byref(K), C.byref(b), rep)
    return K.value, b.value, list(rep)


# ---------------------------------------------------------------- pipeline
class Oracle:
    """Whole-path oracle: scene + display + rig -> V, Psi, pairs, ranges, image."""

    def __init__(self, nthreads: int = 0):
        self._L = lib()
        self._c = self._L.cro_create(nthreads)

    def __del__(self):
        try:
            self._L.cro_destroy(self._c)
        except Exception:
            pass

    @property
    def threads(self) -> int:
        return self._L.cro_threads(self._c)

    def set_tile_pad(self, pad: float):
        """Test knob: grow every tile rectangle of the tile test by pad px."""
        self._L.cro_set_tile_pad(self._c, float(pad))

    def set_scene(self, scene):
        M = int(scene["means"].shape[0])
        deg = int(scene["sh_degree"])
        rc = self._L.cro_set_scene(self._c, M, deg, _f32(scene["means"]).reshape(-1),
                                   _f32(scene["quats"]).reshape(-1),
                                   _f32(scene["scales"]).reshape(-1),
                                   _f32(scene["opacities"]).reshape(-1),
                                   _f32(scene["sh"]).reshape(-1) if M else np.zeros(1, np.float32))
        if rc:
            raise ValueError(f"cro_set_scene: {rc}")
        self.M, self.deg = M, deg

    def constants(self):
        cov = np.zeros((self.M, 6), np.float32)
        tau = np.zeros(self.M, np.float32)
        self._L.cro_get_constants(self._c, cov, tau)
        return cov, tau

    def set_display(self, W, H, N, lens_pitch, slant=None, center_offset=0.0, tan_alpha=None):
        if tan_alpha is not None:
            rc = self._L.cro_set_display_tan(self._c, W, H, N, lens_pitch, tan_alpha,
                                             center_offset)
        else:
            rc = self._L.cro_set_display(self._c, W, H, N, lens_pitch, slant, center_offset)
        if rc:
            raise ValueError(f"cro_set_display: {rc}")
        self.W, self.H, self.N = W, H, N
        self.TX, self.TY = (W + 15) // 16, (H + 15) // 16

    def view_map(self):
        V = np.zeros((self.H, self.W, 3), np.uint8)
        self._L.cro_get_view_map(self._c, V)
        return V

    def remap(self, remap=1):
        psi = np.zeros((self.TY * self.TX, 768), np.uint16)
        self._L.cro_get_remap(self._c, int(remap), psi)
        return psi

    def set_rig(self, cams16, znear=0.01):
        c = _f32(cams16).reshape(-1, 16)
        rc = self._L.cro_set_rig(self._c, c.shape[0], np.ascontiguousarray(c.reshape(-1)), znear)
        if rc:
            raise ValueError(f"cro_set_rig: {rc}")

    def render(self, s=8, row0=0, row1=0, bg=(0, 0, 0), tiles=None, composite=True):
        bgv = _f32(bg).reshape(3)
        if tiles is not None:
            tl = np.ascontiguousarray(tiles, np.int32)
            rc = self._L.cro_render(self._c, s, row0, row1, bgv, tl.ctypes.data, tl.shape[0],
                                    int(composite))
        else:
            rc = self._L.cro_render(self._c, s, row0, row1, bgv, None, 0, int(composite))
        if rc:
            raise ValueError(f"cro_render: {rc}")
        self.s = s
        self.K = self._L.cro_num_clusters(self._c)
        self.bitK = self._L.cro_bit_k(self._c)
        self.row0, self.row1 = row0, (row1 if row1 else self.TY)

    @property
    def num_pairs(self) -> int:
        return self._L.cro_num_pairs(self._c)

    @property
    def num_evals(self) -> int:
        return self._L.cro_num_evals(self._c)

    def pairs(self):
        P = self.num_pairs
        k = np.zeros(P, np.uint64)
        p = np.zeros(P, np.uint32)
        self._L.cro_get_pairs(self._c, k, p)
        return k, p

    def ranges(self):
        n = self.TX * self.TY * self.K
        S = np.zeros(n, np.uint32)
        E = np.zeros(n, np.uint32)
        self._L.cro_get_ranges(self._c, S, E)
        return S.reshape(self.TY * self.TX, self.K), E.reshape(self.TY * self.TX, self.K)

    def image(self):
        y0, y1 = self.row0 * 16, min(self.H, self.row1 * 16)
        img = np.zeros((y1 - y0, self.W, 3), np.float32)
        self._L.cro_get_image(self._c, img)
        return img

    def records(self):
        R = self.K * self.M
        st = np.zeros(R, np.uint8)
        d = np.zeros(R, np.float32)
        cv = np.zeros((R, 4), np.float32)
        cn = np.zeros((R, 3), np.float32)
        col = np.zeros((R, 3), np.float32)
        cnt = np.zeros(R, np.uint32)
        self._L.cro_get_records(self._c, st.ctypes.data, d.ctypes.data, cv.ctypes.data,
                                cn.ctypes.data, col.ctypes.data, cnt.ctypes.data)
        sh = (self.K, self.M)
        return dict(state=st.reshape(sh), depth=d.reshape(sh), cov2d=cv.reshape(sh + (4,)),
                    conic=cn.reshape(sh + (3,)), color=col.reshape(sh + (3,)),
                    count=cnt.reshape(sh))

    def view_frames(self):
        """Per-view frames [N, H, W, 3] of the last full-frame render."""
        out = np.zeros((self.N, self.H, self.W, 3), np.float32)
        if self._L.cro_render_views(self._c, out):
            raise ValueError("cro_render_views needs a full-frame render")
        return out

    def bruteforce(self):
        out = np.zeros((self.H, self.W, 3), np.float32)
        self._L.cro_render_bruteforce(self._c, out)
        return out


def quantize_rgb8(img: np.ndarray) -> np.ndarray:
    """RGB8 = floor(min(max(C,0),1)*255 + 0.5) (round-half-up)."""
    return np.floor(np.clip(img.astype(np.float32), 0.0, 1.0) * np.float32(255.0)
                    + np.float32(0.5)).astype(np.uint8)
