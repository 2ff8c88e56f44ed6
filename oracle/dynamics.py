"""Oracle dynamics (numpy, float64, vectorised over a batch of envs sharing one Model).

Test infrastructure (see oracle/__init__.py).  Restates SPEC.md's kinematics and dynamics
modules with the decisions register in DESIGN.md:
  FK                     SPEC.md:249-257  (compose chain, pose.py:239-249 semantics)
  Jacobian / DLS IK
  ABA (fixed base)       SPEC.md:328-336  (+ CRBA / RNEA cross-check)
  step / drives          SPEC.md:319-327, A-16 (implicit PD through joint armature)
  contacts               SPEC.md:337-345, A-4/A-5/A-6/A-25
  PGS
  integration / limits   SPEC.md:322, 363, A-7/A-8; divergence freeze SPEC.md:323, 367

Spatial vectors are in the WORLD frame about the world origin, motion = (w, v), force =
(n, f); a rigid-body inertia is the triple (m, h = m*c, I_O) with I_O the rotational
inertia about the world origin.
"""

from __future__ import annotations

import numpy as np

from . import se3
from .model import (BODY_ACTOR, BODY_LINK, BODY_STATIC, BOX, CAPSULE, FIXED, PLANE, PRISMATIC,
                    REVOLUTE, SPHERE)


def cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def dot(a, b):
    return np.sum(a * b, axis=-1)


# ----------------------------------------------------------------- kinematics


def joint_motion(model, l, q):
    """Pose of the child link frame relative to the joint frame for joint value(s) q."""
    B = q.shape[0]
    if model.jtype[l] == REVOLUTE:
        h = 0.5 * q
        s = np.sin(h)
        mq = np.stack([np.cos(h), model.axis[l, 0] * s, model.axis[l, 1] * s, model.axis[l, 2] * s], -1)
        return np.zeros((B, 3)), mq
    mp = q[:, None] * model.axis[l][None, :]
    return mp, np.tile([1.0, 0.0, 0.0, 0.0], (B, 1))


def forward_kinematics(model, q):
    """World pose of every link: T_l = T_parent * X_l * Motion(q_l) (roots: T = base pose)."""
    B = q.shape[0]
    P = np.zeros((B, model.L, 3))
    Q = np.zeros((B, model.L, 4))
    for l in range(model.L):
        par = model.parent[l]
        if par < 0:
            P[:, l] = model.org_p[l]
            Q[:, l] = model.org_q[l]
            continue
        jp, jq = se3.compose(P[:, par], Q[:, par], np.broadcast_to(model.org_p[l], (B, 3)),
                             np.broadcast_to(model.org_q[l], (B, 4)))
        if model.jtype[l] == FIXED:
            P[:, l], Q[:, l] = jp, jq
        else:
            mp, mq = joint_motion(model, l, q[:, model.dof_of[l]])
            P[:, l], Q[:, l] = se3.compose(jp, jq, mp, mq)
    return P, Q


def motion_subspace(model, P, Q):
    """S_l (B, L, 6) in world coordinates; zero rows for fixed joints / roots."""
    B = P.shape[0]
    S = np.zeros((B, model.L, 6))
    for l in range(model.L):
        if model.jtype[l] == FIXED:
            continue
        a = se3.qrot(Q[:, l], np.broadcast_to(model.axis[l], (B, 3)))
        if model.jtype[l] == REVOLUTE:
            S[:, l, :3] = a
            S[:, l, 3:] = cross(P[:, l], a)
        else:
            S[:, l, 3:] = a
    return S


def link_world_inertia(model, P, Q):
    """(m, h, I_O) per link: mass, first moment m*c and rotational inertia about the origin."""
    B = P.shape[0]
    R = se3.qmat(Q)  # (B, L, 3, 3)
    c = P + np.einsum("blij,lj->bli", R, model.com)
    Ic = np.einsum("blij,ljk,blmk->blim", R, model.inertia, R)
    m = np.broadcast_to(model.mass, (B, model.L))
    cc = np.einsum("bli,bli->bl", c, c)
    IO = Ic + m[..., None, None] * (cc[..., None, None] * np.eye(3) - np.einsum("bli,blj->blij", c, c))
    return m, m[..., None] * c, IO


def inertia_mul(m, h, IO, V):
    """I * V for V = (w, v): (I_O w + h x v, m v - h x w)."""
    w, v = V[..., :3], V[..., 3:]
    n = np.einsum("...ij,...j->...i", IO, w) + cross(h, v)
    f = m[..., None] * v - cross(h, w)
    return np.concatenate([n, f], -1)


def cross_m(V, U):
    w, v = V[..., :3], V[..., 3:]
    return np.concatenate([cross(w, U[..., :3]), cross(w, U[..., 3:]) + cross(v, U[..., :3])], -1)


def cross_f(V, F):
    w, v = V[..., :3], V[..., 3:]
    return np.concatenate([cross(w, F[..., :3]) + cross(v, F[..., 3:]), cross(w, F[..., 3:])], -1)


def link_velocities(model, S, qd):
    B = qd.shape[0]
    V = np.zeros((B, model.L, 6))
    for l in range(model.L):
        par = model.parent[l]
        if par >= 0:
            V[:, l] = V[:, par]
        if model.jtype[l] != FIXED:
            V[:, l] += S[:, l] * qd[:, model.dof_of[l], None]
    return V


def rnea_bias(model, S, V, inert, qd, gravity, qdd=None):
    """Inverse dynamics tau = M qdd + C (qdd = 0 gives the bias C incl. gravity)."""
    m, h, IO = inert
    B = V.shape[0]
    a = np.zeros((B, model.L, 6))
    g6 = np.concatenate([np.zeros(3), -np.asarray(gravity, np.float64)])
    for l in range(model.L):
        par = model.parent[l]
        a[:, l] = a[:, par] if par >= 0 else g6
        if model.jtype[l] != FIXED:
            d = model.dof_of[l]
            a[:, l] += cross_m(V[:, l], S[:, l] * qd[:, d, None])
            if qdd is not None:
                a[:, l] += S[:, l] * qdd[:, d, None]
    f = inertia_mul(m, h, IO, a) + cross_f(V, inertia_mul(m, h, IO, V))
    tau = np.zeros((B, model.D))
    for l in range(model.L - 1, -1, -1):
        if model.jtype[l] != FIXED:
            tau[:, model.dof_of[l]] = dot(S[:, l], f[:, l])
        par = model.parent[l]
        if par >= 0:
            f[:, par] += f[:, l]
    return tau


def crba(model, S, inert):
    """Joint-space mass matrix via composite rigid bodies (world frame)."""
    m, h, IO = (x.copy() for x in inert)
    m = np.array(m, copy=True)
    B = S.shape[0]
    for l in range(model.L - 1, -1, -1):
        par = model.parent[l]
        if par >= 0:
            m[:, par] += m[:, l]
            h[:, par] += h[:, l]
            IO[:, par] += IO[:, l]
    M = np.zeros((B, model.D, model.D))
    for l in range(model.L):
        if model.jtype[l] == FIXED:
            continue
        i = model.dof_of[l]
        F = inertia_mul(m[:, l], h[:, l], IO[:, l], S[:, l])
        k = l
        while k >= 0:
            if model.jtype[k] != FIXED:
                j = model.dof_of[k]
                M[:, i, j] = M[:, j, i] = dot(S[:, k], F)
            k = model.parent[k]
    return M


def spatial_matrix(m, h, IO):
    B = m.shape[0]
    I6 = np.zeros((B, 6, 6))
    hx = np.zeros((B, 3, 3))
    hx[:, 0, 1], hx[:, 0, 2], hx[:, 1, 0] = -h[:, 2], h[:, 1], h[:, 2]
    hx[:, 1, 2], hx[:, 2, 0], hx[:, 2, 1] = -h[:, 0], -h[:, 1], h[:, 0]
    I6[:, :3, :3] = IO
    I6[:, :3, 3:] = hx
    I6[:, 3:, :3] = np.swapaxes(hx, 1, 2)
    I6[:, 3:, 3:] = m[:, None, None] * np.eye(3)
    return I6


def aba(model, S, V, inert, qd, tau, gravity, armature=None):
    """Featherstone articulated-body algorithm, fixed base.
    `armature` adds to D_i = S^T I^A S (joint-space diagonal), used by the implicit drives."""
    m, h, IO = inert
    B = V.shape[0]
    IA = np.stack([spatial_matrix(m[:, l], h[:, l], IO[:, l]) for l in range(model.L)], 1)
    pA = cross_f(V, inertia_mul(m, h, IO, V))
    c = np.zeros((B, model.L, 6))
    U = np.zeros((B, model.L, 6))
    Dd = np.zeros((B, model.L))
    u = np.zeros((B, model.L))
    for l in range(model.L):
        if model.jtype[l] != FIXED:
            c[:, l] = cross_m(V[:, l], S[:, l] * qd[:, model.dof_of[l], None])
    for l in range(model.L - 1, -1, -1):
        par = model.parent[l]
        if model.jtype[l] != FIXED:
            d = model.dof_of[l]
            U[:, l] = np.einsum("bij,bj->bi", IA[:, l], S[:, l])
            Dd[:, l] = dot(S[:, l], U[:, l]) + (0.0 if armature is None else armature[:, d])
            u[:, l] = tau[:, d] - dot(S[:, l], pA[:, l])
            if par >= 0:
                Ia = IA[:, l] - np.einsum("bi,bj->bij", U[:, l], U[:, l]) / Dd[:, l, None, None]
                pa = pA[:, l] + np.einsum("bij,bj->bi", Ia, c[:, l]) + U[:, l] * (u[:, l] / Dd[:, l])[:, None]
                IA[:, par] += Ia
                pA[:, par] += pa
        elif par >= 0:
            IA[:, par] += IA[:, l]
            pA[:, par] += pA[:, l]
    g6 = np.concatenate([np.zeros(3), -np.asarray(gravity, np.float64)])
    a = np.zeros((B, model.L, 6))
    qdd = np.zeros((B, model.D))
    for l in range(model.L):
        par = model.parent[l]
        ap = a[:, par] if par >= 0 else np.broadcast_to(g6, (B, 6))
        ap = ap + c[:, l]
        if model.jtype[l] != FIXED:
            d = model.dof_of[l]
            qdd[:, d] = (u[:, l] - dot(U[:, l], ap)) / Dd[:, l]
            a[:, l] = ap + S[:, l] * qdd[:, d, None]
        else:
            a[:, l] = ap
    return qdd


def point_jacobian(model, S, link, point):
    """(B, 3, D) linear-velocity Jacobian of a point rigidly attached to `link`."""
    B = S.shape[0]
    J = np.zeros((B, 3, model.D))
    k = link
    while k >= 0:
        if model.jtype[k] != FIXED:
            d = model.dof_of[k]
            J[:, :, d] = S[:, k, 3:] + cross(S[:, k, :3], point)
        k = model.parent[k]
    return J


def geometric_jacobian(model, S, link, point):
    """(B, 6, D): rows (linear xyz, angular xyz) of the frame at `point` on `link`
    (revolute column (z x (p - o), z), prismatic (z, 0))."""
    B = S.shape[0]
    J = np.zeros((B, 6, model.D))
    J[:, :3] = point_jacobian(model, S, link, point)
    k = link
    while k >= 0:
        if model.jtype[k] != FIXED:
            J[:, 3:, model.dof_of[k]] = S[:, k, :3]
        k = model.parent[k]
    return J


def ik_delta(J, twist, lam=0.05):
    """DLS: dq = J^T (J J^T + lam^2 I)^-1 twist via a 6x6 Cholesky."""
    A = np.einsum("bij,bkj->bik", J, J) + (lam * lam) * np.eye(J.shape[1])
    L = np.linalg.cholesky(A)
    y = np.linalg.solve(L, twist[..., None])
    x = np.linalg.solve(np.swapaxes(L, 1, 2), y)
    return np.einsum("bji,bj->bi", J, x[..., 0])
