"""Oracle contact generation (numpy, vectorised over envs) -- test infrastructure.

SPEC.md:337-345: per-env all-pairs broadphase over shapes (no cross-env pairs, no
same-articulation pairs) + narrowphase for sphere/plane, box/plane (<= 4
corners), sphere/sphere, sphere/box, capsule/plane (<= 2 endpoints, A-4).  Unsupported
pairs that pass the broadphase are counted (A-23).

Candidate slots: every pair owns `maxc` fixed slots; a contact exists in a slot when its
depth >= -slop.  The device compacts valid slots in the same order, so slot order ==
contact order (A-5).  Normal points from the second body to the first;
contact point = midpoint between the two surfaces along the normal.
"""

from __future__ import annotations

import numpy as np

from . import se3
from .dynamics import cross, dot
from .model import BODY_ACTOR, BODY_LINK, BOX, CAPSULE, PLANE, SPHERE


def shape_world_poses(model, LP, LQ, AP, AQ):
    """(B, S, 3), (B, S, 4) world poses of every shape slot."""
    B = LP.shape[0]
    P = np.zeros((B, model.S, 3))
    Q = np.zeros((B, model.S, 4))
    for s in range(model.S):
        bt, bi = model.s_btype[s], model.s_body[s]
        if bt == BODY_LINK:
            P[:, s], Q[:, s] = se3.compose(LP[:, bi], LQ[:, bi], np.broadcast_to(model.s_fp[s], (B, 3)),
                                           np.broadcast_to(model.s_fq[s], (B, 4)))
        elif bt == BODY_ACTOR:
            P[:, s], Q[:, s] = AP[:, bi], AQ[:, bi]
        else:
            P[:, s] = model.s_fp[s]
            Q[:, s] = model.s_fq[s]
    return P, Q


def _plane(Pb, Qb):
    n = se3.qrot(Qb, np.broadcast_to([0.0, 0.0, 1.0], Pb.shape))
    return n, Pb


def _sphere_plane(ca, ra, Pb, Qb):
    n, p0 = _plane(Pb, Qb)
    sd = dot(n, ca - p0)
    depth = ra - sd
    sB = ca - sd[:, None] * n
    return [(sB - (0.5 * depth)[:, None] * n, n, depth)]


def _box_plane(Pa, Qa, half, Pb, Qb, slop):
    n, p0 = _plane(Pb, Qb)
    out = []
    depths = []
    for k in range(8):
        sx = half[0] if k & 1 else -half[0]
        sy = half[1] if k & 2 else -half[1]
        sz = half[2] if k & 4 else -half[2]
        corner = Pa + se3.qrot(Qa, np.broadcast_to([sx, sy, sz], Pa.shape))
        sd = dot(n, corner - p0)
        depth = -sd
        sB = corner - sd[:, None] * n
        out.append((sB - (0.5 * depth)[:, None] * n, n, depth))
        depths.append(depth)
    # more than four corners within slop: keep the four deepest (ties -> lower corner index)
    D = np.stack(depths, 1)
    valid = D >= -slop
    many = valid.sum(1) > 4
    if many.any():
        order = np.argsort(-D, axis=1, kind="stable")
        keep = np.zeros_like(valid)
        np.put_along_axis(keep, order[:, :4], True, axis=1)
        drop = many[:, None] & ~keep
        for k in range(8):
            d = out[k][2].copy()
            d[drop[:, k]] = -np.inf
            out[k] = (out[k][0], out[k][1], d)
    return out


def _sphere_sphere(ca, ra, cb, rb):
    d = ca - cb
    dist = np.sqrt(dot(d, d))
    ok = dist > 1e-12
    n = np.where(ok[:, None], d / np.where(ok, dist, 1.0)[:, None], np.array([0.0, 0.0, 1.0]))
    depth = (ra + rb) - dist
    sB = cb + rb * n
    return [(sB - (0.5 * depth)[:, None] * n, n, depth)]


def _sphere_box(ca, ra, Pb, Qb, half):
    local = se3.qrot(se3.qconj(Qb), ca - Pb)
    h = np.asarray(half, np.float64)
    clamped = np.clip(local, -h, h)
    delta = local - clamped
    d2 = dot(delta, delta)
    outside = d2 > 1e-24
    dist = np.sqrt(d2)
    n_out = delta / np.where(outside, dist, 1.0)[:, None]
    pen = h - np.abs(local)
    k = np.argmin(pen, axis=1)
    rows = np.arange(local.shape[0])
    lk = local[rows, k]
    sgn = np.where(lk >= 0.0, 1.0, -1.0)
    n_in = np.zeros_like(local)
    n_in[rows, k] = sgn
    s_in = local.copy()
    s_in[rows, k] = sgn * h[k]
    n_local = np.where(outside[:, None], n_out, n_in)
    s_local = np.where(outside[:, None], clamped, s_in)
    depth = np.where(outside, ra - dist, ra + pen[rows, k])
    n = se3.qrot(Qb, n_local)
    sB = Pb + se3.qrot(Qb, s_local)
    return [(sB - (0.5 * depth)[:, None] * n, n, depth)]


def _capsule_plane(Pa, Qa, r, hl, Pb, Qb):
    n, p0 = _plane(Pb, Qb)
    out = []
    for s in (-hl, hl):
        e = Pa + se3.qrot(Qa, np.broadcast_to([0.0, 0.0, s], Pa.shape))
        sd = dot(n, e - p0)
        depth = r - sd
        sB = e - sd[:, None] * n
        out.append((sB - (0.5 * depth)[:, None] * n, n, depth))
    return out


def narrowphase(model, pair, SP, SQ, slop):
    """List of maxc candidates (point (B,3), normal (B,3) from j to i, depth (B,))."""
    i, j = (pair.j, pair.i) if pair.swap else (pair.i, pair.j)
    ka, kb = pair.kind
    Pa, Qa, Pb, Qb = SP[:, i], SQ[:, i], SP[:, j], SQ[:, j]
    sa, sb = model.s_size[i], model.s_size[j]
    if (ka, kb) == (SPHERE, PLANE):
        cands = _sphere_plane(Pa, sa[0], Pb, Qb)
    elif (ka, kb) == (BOX, PLANE):
        cands = _box_plane(Pa, Qa, sa, Pb, Qb, slop)
    elif (ka, kb) == (SPHERE, SPHERE):
        cands = _sphere_sphere(Pa, sa[0], Pb, sb[0])
    elif (ka, kb) == (SPHERE, BOX):
        cands = _sphere_box(Pa, sa[0], Pb, Qb, sb)
    elif (ka, kb) == (CAPSULE, PLANE):
        cands = _capsule_plane(Pa, Qa, sa[0], sa[1], Pb, Qb)
    else:
        raise AssertionError(pair)
    if pair.swap:
        cands = [(p, -n, d) for (p, n, d) in cands]
    return cands


def broadphase(model, pair, SP, SQ, slop):
    """(B,) bool: bounding spheres (or sphere vs plane half-space) within slop."""
    i, j = pair.i, pair.j
    ki, kj = model.s_kind[i], model.s_kind[j]
    if kj == PLANE or ki == PLANE:
        p_, o_ = (j, i) if kj == PLANE else (i, j)
        n = se3.qrot(SQ[:, p_], np.broadcast_to([0.0, 0.0, 1.0], SP[:, p_].shape))
        return dot(n, SP[:, o_] - SP[:, p_]) <= model.s_radius[o_] + slop
    d = SP[:, i] - SP[:, j]
    return np.sqrt(dot(d, d)) <= (model.s_radius[i] + model.s_radius[j]) + slop


def detect_contacts(model, SP, SQ, slop):
    """Returns dict: slots list of (pair_index, point, normal, depth, valid) and the per-env
    unsupported-pair counter."""
    B = SP.shape[0]
    unsupported = np.zeros(B, np.int64)
    slots = []
    for pi, pair in enumerate(model.pairs):
        near = broadphase(model, pair, SP, SQ, slop)
        if pair.maxc == 0:
            unsupported += near
            continue
        for (p, n, d) in narrowphase(model, pair, SP, SQ, slop):
            valid = near & (d >= -slop)
            slots.append((pi, p, n, d, valid))
    return slots, unsupported


def tangent_basis(n):
    """A-6: e = world axis least aligned with n (ties -> lowest index); t1 = n x e / |.|,
    t2 = n x t1."""
    k = np.argmin(np.abs(n), axis=1)
    e = np.zeros_like(n)
    e[np.arange(n.shape[0]), k] = 1.0
    t1 = cross(n, e)
    t1 = t1 / np.sqrt(dot(t1, t1))[:, None]
    return t1, cross(n, t1)
