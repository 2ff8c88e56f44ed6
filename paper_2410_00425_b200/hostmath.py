"""Host-side (build-time) quaternion helpers for template assembly.

Used only while parsing robot descriptions and packing scene tables on the host -- once
per template, never per step.  Arithmetic order matches the reference pose algebra
(pose.py:31-69) so parsed frames are bit-identical to the reference's templates.
"""

from __future__ import annotations

import math

import numpy as np


def qnormalize(q) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    n = math.sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3])
    u = q / n
    s = 0.0
    for c in u:
        if s == 0.0:
            s = float(np.sign(c))
    if s == 0.0:
        s = 1.0
    return u * s


def qmul(a, b) -> np.ndarray:
    a0, a1, a2, a3 = (float(v) for v in a)
    b0, b1, b2, b3 = (float(v) for v in b)
    return np.array([
        ((a0 * b0 - a1 * b1) - a2 * b2) - a3 * b3,
        ((a0 * b1 + a1 * b0) + a2 * b3) - a3 * b2,
        ((a0 * b2 - a1 * b3) + a2 * b0) + a3 * b1,
        ((a0 * b3 + a1 * b2) - a2 * b1) + a3 * b0,
    ])


def qrotate(q, v) -> np.ndarray:
    w, x, y, z = (float(c) for c in q)
    v0, v1, v2 = (float(c) for c in v)
    t0, t1, t2 = 2.0 * (y * v2 - z * v1), 2.0 * (z * v0 - x * v2), 2.0 * (x * v1 - y * v0)
    return np.array([(v0 + w * t0) + (y * t2 - z * t1),
                     (v1 + w * t1) + (z * t0 - x * t2),
                     (v2 + w * t2) + (x * t1 - y * t0)])


def qmatrix(q) -> np.ndarray:
    w, x, y, z = (float(c) for c in q)
    return np.array([
        [1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)],
        [2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)],
        [2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)],
    ])


def compose(pa, qa, pb, qb):
    """(pa, qa) then (pb, qb): returns (p, q) with q normalized and canonical."""
    p = np.asarray(pa, dtype=np.float64) + qrotate(qa, pb)
    return p, qnormalize(qmul(qa, qb))


def axis_angle_quat(axis, angle: float) -> np.ndarray:
    h = 0.5 * angle
    s = math.sin(h)
    return np.array([math.cos(h), axis[0] * s, axis[1] * s, axis[2] * s])


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """Camera-to-world pose (OpenCV axes: x right, y down, z forward) looking at target."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    if np.linalg.norm(r) < 1e-9:
        r = np.cross(f, np.array([0.0, 1.0, 0.0]))
    r = r / np.linalg.norm(r)
    d = np.cross(f, r)
    m = np.stack([r, d, f], axis=1)  # columns: camera x, y, z in world
    return eye, mat_to_quat(m)


def mat_to_quat(r) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    tr = (r[0, 0] + r[1, 1]) + r[2, 2]
    c = int(np.argmax([tr, r[0, 0], r[1, 1], r[2, 2]]))
    if c == 0:
        s = math.sqrt(1.0 + tr) * 2.0
        q = [0.25 * s, (r[2, 1] - r[1, 2]) / s, (r[0, 2] - r[2, 0]) / s, (r[1, 0] - r[0, 1]) / s]
    elif c == 1:
        s = math.sqrt(1.0 + r[0, 0] - r[1, 1] - r[2, 2]) * 2.0
        q = [(r[2, 1] - r[1, 2]) / s, 0.25 * s, (r[0, 1] + r[1, 0]) / s, (r[0, 2] + r[2, 0]) / s]
    elif c == 2:
        s = math.sqrt(1.0 - r[0, 0] + r[1, 1] - r[2, 2]) * 2.0
        q = [(r[0, 2] - r[2, 0]) / s, (r[0, 1] + r[1, 0]) / s, 0.25 * s, (r[1, 2] + r[2, 1]) / s]
    else:
        s = math.sqrt(1.0 - r[0, 0] - r[1, 1] + r[2, 2]) * 2.0
        q = [(r[1, 0] - r[0, 1]) / s, (r[0, 2] + r[2, 0]) / s, (r[1, 2] + r[2, 1]) / s, 0.25 * s]
    return qnormalize(q)
