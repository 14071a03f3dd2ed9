"""INRIA-3DGS PLY ingestion.

Reads a binary little-endian PLY with vertex properties x, y, z, [nx, ny, nz],
f_dc_0..2, f_rest_0..(3*((d+1)^2-1)-1), opacity (logit), scale_0..2 (log),
rot_0..3 (w, x, y, z) and returns the scene dict the renderer uploads:
opacity = sigmoid(logit), scale = exp(log-scale), quaternions as stored (the
library renormalises), SH in [M][(d+1)^2][3] (INRIA stores f_rest channel-
major: all coefficients of R, then G, then B).  Host-side input plumbing only.
"""
from __future__ import annotations

import numpy as np

_TYPES = {"float": "<f4", "float32": "<f4", "double": "<f8", "uchar": "u1", "uint8": "u1",
          "int": "<i4", "int32": "<i4", "uint": "<u4", "short": "<i2", "ushort": "<u2"}


class PlyError(ValueError):
    pass


def load_ply(path_or_bytes) -> dict:
    data = path_or_bytes if isinstance(path_or_bytes, (bytes, bytearray)) else open(path_or_bytes, "rb").read()
    end = data.find(b"end_header\n")
    if not data.startswith(b"ply") or end < 0:
        raise PlyError("MalformedHeader: not a PLY file")
    header = data[:end].decode("ascii", errors="replace").splitlines()
    fmt = [l for l in header if l.startswith("format")]
    if not fmt or "binary_little_endian" not in fmt[0]:
        raise PlyError("UnsupportedFormat: only binary_little_endian is supported")
    n, props, in_vertex = 0, [], False
    for l in header:
        p = l.split()
        if p[:2] == ["element", "vertex"]:
            n, in_vertex = int(p[2]), True
        elif p and p[0] == "element":
            in_vertex = False
        elif p and p[0] == "property" and in_vertex:
            if p[1] == "list":
                raise PlyError("UnsupportedFormat: list properties in vertex element")
            props.append((p[2], _TYPES[p[1]]))
    dt = np.dtype(props)
    body = data[end + len(b"end_header\n"):]
    if len(body) < n * dt.itemsize:
        raise PlyError("TruncatedBody")
    v = np.frombuffer(body, dt, count=n)
    names = set(v.dtype.names)
    need = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1",
            "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    missing = [q for q in need if q not in names]
    if missing:
        raise PlyError(f"MalformedHeader: missing {missing}")
    nrest = len([q for q in names if q.startswith("f_rest_")])
    nc = nrest // 3 + 1
    deg = int(round(np.sqrt(nc))) - 1
    if (deg + 1) ** 2 != nc or deg > 3:
        raise PlyError(f"MalformedHeader: {nrest} f_rest values is not a SH degree <= 3")
    f = lambda q: v[q].astype(np.float32)
    means = np.stack([f("x"), f("y"), f("z")], 1)
    sh = np.zeros((n, nc, 3), np.float32)
    sh[:, 0, :] = np.stack([f("f_dc_0"), f("f_dc_1"), f("f_dc_2")], 1)
    for ch in range(3):
        for m in range(1, nc):
            sh[:, m, ch] = f(f"f_rest_{ch * (nc - 1) + (m - 1)}")
    scene = dict(means=means,
                 quats=np.stack([f("rot_0"), f("rot_1"), f("rot_2"), f("rot_3")], 1),
                 scales=np.exp(np.stack([f("scale_0"), f("scale_1"), f("scale_2")], 1)).astype(np.float32),
                 opacities=(1.0 / (1.0 + np.exp(-f("opacity").astype(np.float64)))).astype(np.float32),
                 sh=sh, sh_degree=deg)
    for k_, a in scene.items():
        if isinstance(a, np.ndarray) and not np.all(np.isfinite(a)):
            raise PlyError(f"NonFiniteValue in {k_}")
    return scene


def save_ply(scene: dict, path=None) -> bytes:
    """Inverse of load_ply (for round trips and exporting synthetic scenes)."""
    M = scene["means"].shape[0]
    nc = (scene["sh_degree"] + 1) ** 2
    cols = [("x", scene["means"][:, 0]), ("y", scene["means"][:, 1]), ("z", scene["means"][:, 2])]
    cols += [(f"f_dc_{c}", scene["sh"][:, 0, c]) for c in range(3)]
    cols += [(f"f_rest_{c * (nc - 1) + (m - 1)}", scene["sh"][:, m, c])
             for c in range(3) for m in range(1, nc)]
    o = np.clip(scene["opacities"].astype(np.float64), 1e-7, 1 - 1e-7)
    cols.append(("opacity", np.log(o / (1 - o))))
    cols += [(f"scale_{c}", np.log(scene["scales"][:, c])) for c in range(3)]
    cols += [(f"rot_{c}", scene["quats"][:, c]) for c in range(4)]
    dt = np.dtype([(nme, "<f4") for nme, _ in cols])
    arr = np.zeros(M, dt)
    for nme, val in cols:
        arr[nme] = val
    head = ("ply\nformat binary_little_endian 1.0\nelement vertex %d\n" % M +
            "".join(f"property float {nme}\n" for nme, _ in cols) + "end_header\n").encode()
    blob = head + arr.tobytes()
    if path:
        open(path, "wb").write(blob)
    return blob
