"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds NO arithmetic of the method: it only draws Gaussian scenes,
builds camera rigs (look-at cameras on an orbit arc) and names the display
configurations of BASELINE.json.  Both the CUDA path and the CPU oracle take
its outputs as inputs.  Recipes: DESIGN.md §4.

Layouts (all float32, C-contiguous):
  means     [M, 3]     world position
  quats     [M, 4]     (w, x, y, z), not necessarily normalised
  scales    [M, 3]     per-axis standard deviation (linear, > 0)
  opacities [M]        post-sigmoid, in [0, 1]
  sh        [M, (deg+1)^2, 3]  coefficient-major, channel-minor (gsplat layout)
  cameras   [N, 16]    R[9] (world->camera, row-major, OpenCV axes), t[3], fx, fy, cx, cy
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GENERATOR_VERSION = "scene_gen v1"

# DC coefficient scale: a palette value p in [0.1, 0.9] is stored as (p-0.5)*3.5449
# so that 3DGS-convention DC colours land near p (generator choice, not the method).
_DC_SCALE = 3.5449077018110318


def _unit_quats(rng, n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def _quat_from_axes(t1, t2, nrm):
    """Quaternion (w,x,y,z) of the rotation whose columns are (t1, t2, nrm)."""
    m = np.stack([t1, t2, nrm], axis=2)  # [n,3,3], columns
    n = m.shape[0]
    q = np.zeros((n, 4))
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    # Shepperd's method, branch per row
    c0 = tr > 0
    s = np.sqrt(np.maximum(tr + 1.0, 1e-12)) * 2
    q[c0, 0] = 0.25 * s[c0]
    q[c0, 1] = (m[c0, 2, 1] - m[c0, 1, 2]) / s[c0]
    q[c0, 2] = (m[c0, 0, 2] - m[c0, 2, 0]) / s[c0]
    q[c0, 3] = (m[c0, 1, 0] - m[c0, 0, 1]) / s[c0]
    rest = ~c0
    d = np.stack([m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]], axis=1)
    am = np.argmax(d, axis=1)
    for a in range(3):
        sel = rest & (am == a)
        if not np.any(sel):
            continue
        b, c = (a + 1) % 3, (a + 2) % 3
        s2 = np.sqrt(np.maximum(1.0 + m[sel, a, a] - m[sel, b, b] - m[sel, c, c], 1e-12)) * 2
        q[sel, 0] = (m[sel, c, b] - m[sel, b, c]) / s2
        q[sel, 1 + a] = 0.25 * s2
        q[sel, 1 + b] = (m[sel, b, a] + m[sel, a, b]) / s2
        q[sel, 1 + c] = (m[sel, c, a] + m[sel, a, c]) / s2
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _tangents(nrm, rng):
    """Random tangent frame (t1, t2) orthogonal to unit normals nrm."""
    a = rng.standard_normal(nrm.shape)
    t1 = a - np.sum(a * nrm, axis=1, keepdims=True) * nrm
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(nrm, t1)
    return t1, t2


def _palette(pos, seed):
    """Smooth position-hash palette in [0.1, 0.9]^3."""
    ph = np.random.default_rng(seed + 7).uniform(0, 2 * np.pi, (3, 3))
    fr = np.array([1.7, 2.3, 3.1])
    c = np.empty((pos.shape[0], 3))
    for ch in range(3):
        v = (np.sin(fr[ch] * pos[:, 0] + ph[ch, 0]) * np.sin(fr[(ch + 1) % 3] * pos[:, 1] + ph[ch, 1])
             + np.sin(fr[(ch + 2) % 3] * pos[:, 2] + ph[ch, 2]))
        c[:, ch] = 0.5 + 0.2 * v
    return np.clip(c, 0.1, 0.9)


def _sh_coeffs(rng, pos, deg, seed):
    n = pos.shape[0]
    nc = (deg + 1) ** 2
    sh = np.zeros((n, nc, 3))
    sh[:, 0, :] = (_palette(pos, seed) - 0.5) * _DC_SCALE
    m = 1
    for l in range(1, deg + 1):
        cnt = 2 * l + 1
        sh[:, m:m + cnt, :] = rng.normal(0.0, 0.03 / l, (n, cnt, 3))
        m += cnt
    return sh


def _opacity(rng, n):
    hi = rng.random(n) < 0.65
    return np.where(hi, rng.uniform(0.7, 1.0, n), rng.uniform(0.02, 0.3, n))


def random_scene(M: int, sh_degree: int = 0, seed: int = 0, extent: float = 1.0,
                 scale_median: float = 0.03) -> dict:
    """Config A scene: means uniform in [-extent, extent]^3, lognormal scales,
    random unit quaternions, opacity U[0.05, 1], random DC colour."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(-extent, extent, (M, 3))
    scales = np.exp(rng.normal(math.log(scale_median), 0.5, (M, 3)))
    quats = _unit_quats(rng, M)
    opac = rng.uniform(0.05, 1.0, M)
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((M, nc, 3))
    sh[:, 0, :] = rng.uniform(-1.5, 1.5, (M, 3))
    for m in range(1, nc):
        sh[:, m, :] = rng.normal(0.0, 0.05, (M, 3))
    return _pack(means, quats, scales, opac, sh, sh_degree)


def scene_gen_v1(M: int, sh_degree: int = 3, seed: int = 0) -> dict:
    """Mip-NeRF-360-shaped synthetic scene ('scene_gen v1'):
    55% object surfaces (8 ellipsoids), 30% ground disc, 15% background shell."""
    rng = np.random.default_rng(seed)
    n_obj = int(round(M * 0.55))
    n_gnd = int(round(M * 0.30))
    n_bkg = M - n_obj - n_gnd
    # object: surfaces of 8 random ellipsoids
    centres = rng.uniform(-0.7, 0.7, (8, 3))
    centres[:, 1] = rng.uniform(-0.3, 0.05, 8)
    radii = rng.uniform(0.2, 0.8, (8, 3))
    which = rng.integers(0, 8, n_obj)
    u = rng.standard_normal((n_obj, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    p_obj = centres[which] + radii[which] * u
    n_obj_v = u / radii[which] ** 2
    n_obj_v /= np.linalg.norm(n_obj_v, axis=1, keepdims=True)
    t1, t2 = _tangents(n_obj_v, rng)
    q_obj = _quat_from_axes(t1, t2, n_obj_v)
    s_obj = np.exp(rng.normal(math.log(0.003), 0.5, (n_obj, 3)))
    s_obj[:, 2] *= rng.uniform(0.1, 0.3, n_obj)
    # ground: disc r <= 6 at y = -1
    r = 6.0 * np.sqrt(rng.random(n_gnd))
    th = rng.uniform(0, 2 * np.pi, n_gnd)
    p_gnd = np.stack([r * np.cos(th), -1.0 + rng.normal(0, 0.05, n_gnd), r * np.sin(th)], 1)
    n_gnd_v = np.tile(np.array([0.0, 1.0, 0.0]), (n_gnd, 1))
    g1, g2 = _tangents(n_gnd_v, rng)
    q_gnd = _quat_from_axes(g1, g2, n_gnd_v)
    s_gnd = np.exp(rng.normal(math.log(0.005), 0.5, (n_gnd, 3)))
    s_gnd[:, 2] *= 0.2
    # background: sphere shell r in U[15, 40]
    d = rng.standard_normal((n_bkg, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p_bkg = d * rng.uniform(15, 40, (n_bkg, 1))
    q_bkg = _unit_quats(rng, n_bkg)
    s_bkg = np.exp(rng.normal(math.log(0.08), 0.6, (n_bkg, 3)))

    means = np.concatenate([p_obj, p_gnd, p_bkg])
    quats = np.concatenate([q_obj, q_gnd, q_bkg])
    scales = np.concatenate([s_obj, s_gnd, s_bkg])
    opac = _opacity(rng, M)
    sh = _sh_coeffs(rng, means, sh_degree, seed)
    perm = rng.permutation(M)  # interleave components (no index/position correlation)
    return _pack(means[perm], quats[perm], scales[perm], opac[perm], sh[perm], sh_degree)


def _pack(means, quats, scales, opac, sh, deg):
    return dict(means=np.ascontiguousarray(means, np.float32),
                quats=np.ascontiguousarray(quats, np.float32),
                scales=np.ascontiguousarray(scales, np.float32),
                opacities=np.ascontiguousarray(opac, np.float32),
                sh=np.ascontiguousarray(sh, np.float32), sh_degree=int(deg))


def empty_scene(sh_degree=0):
    nc = (sh_degree + 1) ** 2
    return _pack(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                 np.zeros((0, nc, 3)), sh_degree)


def look_at_camera(C, target, up, fx, fy, cx, cy):
    """World->camera (R, t) for a pinhole at C looking at target, OpenCV axes
    (x right, y down, z forward)."""
    C = np.asarray(C, np.float64)
    f = np.asarray(target, np.float64) - C
    f /= np.linalg.norm(f)
    x = np.cross(f, np.asarray(up, np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f])
    t = -R @ C
    return np.concatenate([R.reshape(9), t, [fx, fy, cx, cy]]).astype(np.float32)


def orbit_rig(N: int, cone_deg: float, W: int, H: int, radius: float = 4.0,
              height: float = 0.8, fov_y_deg: float = 40.0, look_at=(0.0, 0.0, 0.0),
              up=(0.0, 1.0, 0.0), yaw_deg: float = 0.0, pitch_deg: float = 0.0) -> np.ndarray:
    """N inward-looking cameras on a horizontal arc of `cone_deg` (53 deg);
    view 0 at -cone/2 (leftmost seen from +z).  Returns [N, 16] float32."""
    fy = H / (2.0 * math.tan(math.radians(fov_y_deg) / 2.0))
    fx = fy
    cams = np.zeros((N, 16), np.float32)
    la = np.asarray(look_at, np.float64)
    for j in range(N):
        th = math.radians(yaw_deg + (-cone_deg / 2.0 + (cone_deg * j / (N - 1) if N > 1 else
                                                         cone_deg / 2.0)))
        ph = math.radians(pitch_deg)
        C = la + np.array([radius * math.sin(th) * math.cos(ph),
                           height + radius * math.sin(ph),
                           radius * math.cos(th) * math.cos(ph)])
        cams[j] = look_at_camera(C, la, up, fx, fy, W / 2.0, H / 2.0)
    return cams


def identical_rig(N: int, W: int, H: int, **kw) -> np.ndarray:
    """All N cameras at one pose (degenerate rig used by the reuse invariant)."""
    c = orbit_rig(1, 0.0, W, H, **kw)
    return np.repeat(c, N, axis=0)


@dataclass
class Config:
    name: str
    M: int
    sh_degree: int
    N: int
    W: int
    H: int
    lens_pitch: float
    slant: float          # radians
    center_offset: float
    view_cone: float      # degrees
    cluster_size: int
    scene: str            # "random" | "scene_gen_v1"
    seed: int = 0
    rig: dict = field(default_factory=dict)
    gpus: int = 1

    def make_scene(self):
        if self.scene == "random":
            return random_scene(self.M, self.sh_degree, self.seed)
        return scene_gen_v1(self.M, self.sh_degree, self.seed)

    def make_rig(self, **over):
        kw = dict(self.rig)
        kw.update(over)
        return orbit_rig(self.N, self.view_cone, self.W, self.H, **kw)

    def display(self):
        return dict(width=self.W, height=self.H, num_views=self.N, lens_pitch=self.lens_pitch,
                    slant=self.slant, center_offset=self.center_offset,
                    view_cone=self.view_cone)


_SLANT_LG = math.atan(0.1852)
# BASELINE.json configs[0..4] (display table in §8d)
CONFIGS = {
    "A": Config("A", 10_000, 0, 8, 256, 144, 12.5, math.atan(0.25), 1.5, 8.0, 8, "random", 0,
                dict(radius=3.0, height=0.0, fov_y_deg=50.0)),
    "B": Config("B", 1_000_000, 3, 45, 3840, 2160, 19.6153, _SLANT_LG, 7.3, 53.0, 8,
                "scene_gen_v1", 0),
    "C": Config("C", 3_000_000, 3, 100, 3840, 2160, 19.6153, _SLANT_LG, 7.3, 53.0, 8,
                "scene_gen_v1", 0),
    "D": Config("D", 6_000_000, 3, 100, 7680, 4320, 19.6153, _SLANT_LG, 7.3, 53.0, 8,
                "scene_gen_v1", 0, gpus=8),
    "E": Config("E", 3_000_000, 3, 45, 3840, 2160, 19.6153, _SLANT_LG, 7.3, 53.0, 8,
                "scene_gen_v1", 0, gpus=8),
    # the paper's own display setups on the
    # 3M-Gaussian synthetic scene: 63-view 1440x2560 portrait (s=16) and
    # 71-view 3840x2160 landscape (s=18); lens parameters are unpublished
    # (S:206), so the Looking-Glass-style values above are reused.
    "P2K": Config("P2K", 3_000_000, 3, 63, 1440, 2560, 19.6153, _SLANT_LG, 7.3, 53.0, 16,
                  "scene_gen_v1", 0),
    "P4K": Config("P4K", 3_000_000, 3, 71, 3840, 2160, 19.6153, _SLANT_LG, 7.3, 53.0, 18,
                  "scene_gen_v1", 0),
}


def head_tracked_poses(n: int = 256, seed: int = 1):
    """Config E poses: yaw U[-15,15] deg, pitch U[-5,5] deg, radius 4*U[0.9,1.1]."""
    rng = np.random.default_rng(seed)
    return [dict(yaw_deg=float(rng.uniform(-15, 15)), pitch_deg=float(rng.uniform(-5, 5)),
                 radius=float(4.0 * rng.uniform(0.9, 1.1))) for _ in range(n)]
