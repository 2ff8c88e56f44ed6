"""Build-time tessellation of the primitive shapes for the batched rasterizer.

SPEC.md:461 fixes the cached unit-mesh sizes: sphere 320 triangles, box 12, capsule 512,
cylinder 64. DESIGN.md A-9/A-11 add the ground plane, drawn as a finite grid. Meshes are
generated once per distinct env layout on the host, in float64, then scaled by the shape
size and rounded to float32. The rasterizer (csrc/raster.cu) and the CPU oracle
(oracle/raster.py) consume exactly these arrays.

Conventions:
- Vertices are in the shape's local frame. Capsule and cylinder axes are local z
  (assets.py capsule/cylinder).
- Triangles are wound counter-clockwise around their outward normal.
"""

from __future__ import annotations

import math

import numpy as np

SEGMENTS = 16          # around capsule / cylinder axes
CAPSULE_RINGS = 6      # latitude rings per hemisphere (equator included)
CAPSULE_BANDS = 5      # segments along the capsule's cylindrical side (short triangles, small
                       # bounding boxes): 2 * (16 + 32 * 5) + 32 * 5 = 512 triangles
GROUND_EXTENT = 1.0    # ground grid half-extent, m
GROUND_CELLS = 8       # ground grid cells per side


def _icosphere(level: int = 2):
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.array(p, np.float64) / np.linalg.norm(p) for p in v]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
             (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return np.array(verts), np.array(faces, np.int32)


def _box():
    v = np.array([[(1 if k & 1 else -1), (1 if k & 2 else -1), (1 if k & 4 else -1)] for k in range(8)], np.float64)
    f = [(0, 2, 3), (0, 3, 1),   # -z
         (4, 5, 7), (4, 7, 6),   # +z
         (0, 1, 5), (0, 5, 4),   # -y
         (2, 6, 7), (2, 7, 3),   # +y
         (0, 4, 6), (0, 6, 2),   # -x
         (1, 3, 7), (1, 7, 5)]   # +x
    return v, np.array(f, np.int32)


def _capsule(r: float, hl: float):
    S, K = SEGMENTS, CAPSULE_RINGS
    verts = [(0.0, 0.0, hl + r)]  # top pole
    for k in range(1, K + 1):     # top hemisphere rings, ring K = equator
        th = (math.pi / 2) * k / K
        for s in range(S):
            ph = 2 * math.pi * s / S
            verts.append((r * math.sin(th) * math.cos(ph), r * math.sin(th) * math.sin(ph), hl + r * math.cos(th)))
    for b in range(1, CAPSULE_BANDS):  # intermediate rings along the side
        z = hl - 2.0 * hl * b / CAPSULE_BANDS
        for s in range(S):
            ph = 2 * math.pi * s / S
            verts.append((r * math.cos(ph), r * math.sin(ph), z))
    for k in range(K, 0, -1):     # bottom hemisphere rings, equator first
        th = (math.pi / 2) * k / K
        for s in range(S):
            ph = 2 * math.pi * s / S
            verts.append((r * math.sin(th) * math.cos(ph), r * math.sin(th) * math.sin(ph), -hl - r * math.cos(th)))
    verts.append((0.0, 0.0, -hl - r))  # bottom pole
    nring = 2 * K + CAPSULE_BANDS - 1
    ring = lambda k, s: 1 + k * S + (s % S)  # noqa: E731
    f = []
    for s in range(S):
        f.append((0, ring(0, s), ring(0, s + 1)))
    for k in range(nring - 1):
        for s in range(S):
            a, b, c, d = ring(k, s), ring(k, s + 1), ring(k + 1, s), ring(k + 1, s + 1)
            f += [(a, c, d), (a, d, b)]
    bot = len(verts) - 1
    for s in range(S):
        f.append((bot, ring(nring - 1, s + 1), ring(nring - 1, s)))
    return np.array(verts, np.float64), np.array(f, np.int32)


def _cylinder(r: float, hl: float):
    S = SEGMENTS
    verts = []
    for z in (hl, -hl):
        for s in range(S):
            ph = 2 * math.pi * s / S
            verts.append((r * math.cos(ph), r * math.sin(ph), z))
    verts += [(0.0, 0.0, hl), (0.0, 0.0, -hl)]
    top, bot = 2 * S, 2 * S + 1
    f = []
    for s in range(S):
        a, b = s, (s + 1) % S
        c, d = S + s, S + (s + 1) % S
        f += [(a, c, d), (a, d, b)]
        f.append((top, a, b))
        f.append((bot, d, c))
    return np.array(verts, np.float64), np.array(f, np.int32)


def _ground():
    n, e = GROUND_CELLS, GROUND_EXTENT
    xs = np.linspace(-e, e, n + 1)
    verts = [(x, y, 0.0) for y in xs for x in xs]
    f = []
    for j in range(n):
        for i in range(n):
            a = j * (n + 1) + i
            b, c, d = a + 1, a + n + 1, a + n + 2
            f += [(a, b, d), (a, d, c)]
    return np.array(verts, np.float64), np.array(f, np.int32)


def shape_mesh(kind: str, size) -> tuple:
    """(verts float32 (V,3), tris int32 (T,3)) of one shape in its local frame."""
    if kind == "sphere":
        v, f = _icosphere(2)
        v = v * size[0]
    elif kind == "box":
        v, f = _box()
        v = v * np.asarray(size[:3], np.float64)
    elif kind == "capsule":
        v, f = _capsule(size[0], size[1])
    elif kind == "cylinder":
        v, f = _cylinder(size[0], size[1])
    elif kind == "plane":
        v, f = _ground()
    else:
        raise ValueError(f"no tessellation for shape kind {kind!r}")
    return v.astype(np.float32), f.astype(np.int32)


def model_mesh(shapes) -> dict:
    """Concatenate the meshes of one model's shape slots (scene.PackedModel.shapes order).
    Returns verts (V,3) f32, vert_shape (V,), tris (T,3) model-local, tri_shape (T,)."""
    vs, vsh, ts, tsh = [], [], [], []
    base = 0
    for s, sh in enumerate(shapes):
        v, f = shape_mesh(sh["kind"], sh["size"])
        vs.append(v)
        vsh.append(np.full(len(v), s, np.int32))
        ts.append(f + base)
        tsh.append(np.full(len(f), s, np.int32))
        base += len(v)
    return {"verts": np.concatenate(vs) if vs else np.zeros((0, 3), np.float32),
            "vert_shape": np.concatenate(vsh) if vsh else np.zeros(0, np.int32),
            "tris": np.concatenate(ts) if ts else np.zeros((0, 3), np.int32),
            "tri_shape": np.concatenate(tsh) if tsh else np.zeros(0, np.int32)}
