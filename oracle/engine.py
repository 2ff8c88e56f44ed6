"""Oracle step: controller -> substeps (drives, ABA-equivalent dynamics, contacts, PGS,
integration, limits, divergence) -> FK cache.  Test infrastructure (oracle/__init__.py).

Vectorised over a batch of B envs that share one Model.  Follows SPEC.md:319-327 (step),
SPEC.md:346-354 (PGS), SPEC.md:402-410 (controllers) with DESIGN.md's decisions:
  A-16  PD drives with a target position AND a target velocity (DriveTargets):
        tau = kp(q* - q) + kd(qd* - qd), the gains taken "per unit inertia scale"
        (SPEC.md:427): Kp = kp * m, Kd = kd * m with m = M_ii(q) the joint-space inertia of the
        dof, so kd = 2 sqrt(kp) is critical damping for every dof whatever its inertia.  The
        drive is evaluated implicitly at the end-of-substep velocity (stable at kp = 1000,
        dt = 1/120):
          (M + diag(dt*(Kd + damping) + dt^2*Kp)) qdd
              = clamp(Kp(q* - q - dt*qd) + Kd(qd* - qd), +-limit) - damping*qd - C(q, qd)
  A-7   joint limits: clamp after integration, zero the velocity into the limit
  A-8   free bodies: q <- normalize(q + dt/2 (0,w) q) with the (post-contact) velocity w, then
        the world angular momentum is carried to the new orientation:
        w' = I_w(q')^-1 I_w(q) w -- torque-free rotation conserves L = I_w w exactly
        (SPEC.md:358), the gyroscopic effect included
  bias  normal-row target: beta*(d-slop)/dt if d > slop; 0 if 0 <= d <= slop; d/dt if d < 0
        (speculative); velocity iterations keep only the speculative part
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import se3
from .contacts import detect_contacts, shape_world_poses, tangent_basis
from .dynamics import (aba, crba, cross, dot, forward_kinematics, geometric_jacobian, ik_delta,
                       link_velocities, link_world_inertia, motion_subspace, point_jacobian, rnea_bias)
from .model import BODY_ACTOR, BODY_LINK


@dataclass
class SimConfig:
    sim_freq: int = 120
    control_freq: int = 60
    solver_pos_iters: int = 4
    solver_vel_iters: int = 0
    gravity: tuple = (0.0, 0.0, -9.81)
    friction_coeff: float = 1.0
    restitution: float = 0.0
    penetration_slop: float = 5e-4
    baumgarte_beta: float = 0.2

    @property
    def substeps(self) -> int:
        return self.sim_freq // self.control_freq

    @property
    def dt(self) -> float:
        return 1.0 / self.sim_freq


@dataclass
class Drives:
    """Per-dof drive parameters (D,) + per-env targets (B, D)."""

    kp: np.ndarray
    kd: np.ndarray
    force_limit: np.ndarray
    target: np.ndarray = None
    target_vel: np.ndarray = None


@dataclass
class State:
    q: np.ndarray
    qd: np.ndarray
    ap: np.ndarray
    aq: np.ndarray
    av: np.ndarray
    aw: np.ndarray
    diverged: np.ndarray = None
    contacts: list = field(default_factory=list)
    unsupported: np.ndarray = None

    def copy(self):
        return State(self.q.copy(), self.qd.copy(), self.ap.copy(), self.aq.copy(), self.av.copy(),
                     self.aw.copy(), None if self.diverged is None else self.diverged.copy())


def actor_world_inertia(model, aq):
    R = se3.qmat(aq)  # (B, A, 3, 3)
    Iw = np.einsum("baij,aj,bakj->baik", R, model.actor_inertia, R)
    Iw_inv = np.einsum("baij,aj,bakj->baik", R, 1.0 / model.actor_inertia, R) if model.A else Iw
    return Iw, Iw_inv


def substep(model, st: State, drv: Drives, cfg: SimConfig, want_contacts=False):
    dt = cfg.dt
    B = st.q.shape[0]
    g = np.asarray(cfg.gravity, np.float64)
    q, qd = st.q, st.qd
    # ---- articulation forward dynamics (CRBA/RNEA form; ABA cross-checked in tests)
    LP, LQ = forward_kinematics(model, q)
    S = motion_subspace(model, LP, LQ)
    V = link_velocities(model, S, qd)
    inert = link_world_inertia(model, LP, LQ)
    D = model.D
    if D:
        C = rnea_bias(model, S, V, inert, qd, g)
        M = crba(model, S, inert)
        m_ii = np.diagonal(M, axis1=1, axis2=2)           # inertia scale of each dof (A-16)
        Kp, Kd = drv.kp * m_ii, drv.kd * m_ii
        tv = np.zeros_like(q) if drv.target_vel is None else drv.target_vel
        arm = dt * (Kd + model.damping) + (dt * dt) * Kp
        Mt = M + arm[:, :, None] * np.eye(D)[None]
        tau = np.clip(Kp * ((drv.target - q) - dt * qd) + Kd * (tv - qd),
                      -drv.force_limit, drv.force_limit) - model.damping * qd
        qdd = np.linalg.solve(Mt, (tau - C)[..., None])[..., 0]
        Mt_inv = np.linalg.inv(Mt)
    else:
        qdd = np.zeros((B, 0))
        Mt_inv = np.zeros((B, 0, 0))
    u_q = qd + dt * qdd
    # ---- free bodies
    Iw, Iw_inv = actor_world_inertia(model, st.aq)
    u_w = st.aw.copy()
    u_v = st.av + dt * g
    # ---- contacts at start-of-substep positions
    SP, SQ = shape_world_poses(model, LP, LQ, st.ap, st.aq)
    slots, unsupported = detect_contacts(model, SP, SQ, cfg.penetration_slop)
    rows = []
    for (pi, P, n, depth, valid) in slots:
        pair = model.pairs[pi]
        t1, t2 = tangent_basis(n)
        crow = []
        for e in (n, t1, t2):
            Ja = np.zeros((B, D))
            act = []
            for slot, sgn in ((pair.i, 1.0), (pair.j, -1.0)):
                bt, bi = model.s_btype[slot], model.s_body[slot]
                if bt == BODY_LINK and not model.grounded[bi]:
                    Jp = point_jacobian(model, S, bi, P)
                    Ja += sgn * np.einsum("bkd,bk->bd", Jp, e)
                elif bt == BODY_ACTOR:
                    r = P - st.ap[:, bi]
                    act.append((bi, sgn * e, sgn * cross(r, e)))
            Wa = np.einsum("bij,bj->bi", Mt_inv, Ja)
            K = dot(Ja, Wa)
            acts = []
            for (a, Jv, Jw) in act:
                Ww = np.einsum("bij,bj->bi", Iw_inv[:, a], Jw)
                K = K + (dot(Jv, Jv) / model.actor_mass[a] + dot(Jw, Ww))
                acts.append((a, Jv, Jw, Jv / model.actor_mass[a], Ww))
            crow.append((Ja, Wa, acts, K))
        d = depth
        bias = np.where(d > cfg.penetration_slop, cfg.baumgarte_beta * (d - cfg.penetration_slop) / dt,
                        np.where(d >= 0.0, 0.0, d / dt))
        spec = np.where(d < 0.0, d / dt, 0.0)
        rows.append((crow, bias, spec, valid))
    # ---- projected Gauss-Seidel, per-env sequential sweeps
    lam = [np.zeros((B, 3)) for _ in rows]
    mu = cfg.friction_coeff
    for it in range(cfg.solver_pos_iters + cfg.solver_vel_iters):
        pos_phase = it < cfg.solver_pos_iters
        for c, (crow, bias, spec, valid) in enumerate(rows):
            for r in range(3):
                Ja, Wa, acts, K = crow[r]
                vrow = dot(Ja, u_q)
                for (a, Jv, Jw, _, _) in acts:
                    vrow = vrow + (dot(Jv, u_v[:, a]) + dot(Jw, u_w[:, a]))
                ok = valid & (K > 1e-12)
                Ks = np.where(ok, K, 1.0)
                old = lam[c][:, r]
                if r == 0:
                    tgt = bias if pos_phase else spec
                    new = np.maximum(old + (tgt - vrow) / Ks, 0.0)
                else:
                    bound = mu * lam[c][:, 0]
                    new = np.clip(old + (0.0 - vrow) / Ks, -bound, bound)
                delta = np.where(ok, new - old, 0.0)
                lam[c][:, r] = np.where(ok, new, old)
                u_q = u_q + delta[:, None] * Wa
                for (a, _, _, Wv, Ww) in acts:
                    u_v[:, a] += delta[:, None] * Wv
                    u_w[:, a] += delta[:, None] * Ww
    # ---- integrate, limits
    q1 = q + dt * u_q
    lo, hi = model.lower, model.upper
    below, above = q1 < lo, q1 > hi
    q1 = np.where(below, lo, np.where(above, hi, q1))
    qd1 = np.where(below, np.maximum(u_q, 0.0), np.where(above, np.minimum(u_q, 0.0), u_q))
    ap1 = st.ap + dt * u_v
    if model.A:
        wq = np.concatenate([np.zeros(u_w.shape[:-1] + (1,)), u_w], -1)
        aq1 = se3.qnorm(st.aq + (0.5 * dt) * se3.qmul(wq, st.aq))
        # carry the angular momentum to the new orientation (A-8)
        _, Iw1_inv = actor_world_inertia(model, aq1)
        u_w = np.einsum("baij,baj->bai", Iw1_inv, np.einsum("baij,baj->bai", Iw, u_w))
    else:
        aq1 = st.aq.copy()
    finite = (np.isfinite(q1).all(1) & np.isfinite(qd1).all(1)
              & np.isfinite(ap1).reshape(B, -1).all(1) & np.isfinite(aq1).reshape(B, -1).all(1)
              & np.isfinite(u_v).reshape(B, -1).all(1) & np.isfinite(u_w).reshape(B, -1).all(1))
    frozen = st.diverged.astype(bool) if st.diverged is not None else np.zeros(B, bool)
    take = finite & ~frozen
    out = State(np.where(take[:, None], q1, q), np.where(take[:, None], qd1, qd),
                np.where(take[:, None, None], ap1, st.ap), np.where(take[:, None, None], aq1, st.aq),
                np.where(take[:, None, None], u_v, st.av), np.where(take[:, None, None], u_w, st.aw),
                (frozen | ~finite).astype(np.uint8))
    out.unsupported = unsupported
    if want_contacts:
        out.contacts = [(model.pairs[pi].i, model.pairs[pi].j, P, n, d, v) for (pi, P, n, d, v) in slots]
    return out


def aba_qdd(model, q, qd, tau, gravity, armature=None):
    """ABA on its own: used by the KAT and the CRBA/RNEA cross-check."""
    LP, LQ = forward_kinematics(model, q)
    S = motion_subspace(model, LP, LQ)
    V = link_velocities(model, S, qd)
    return aba(model, S, V, link_world_inertia(model, LP, LQ), qd, tau, gravity, armature)


def crba_rnea_qdd(model, q, qd, tau, gravity):
    LP, LQ = forward_kinematics(model, q)
    S = motion_subspace(model, LP, LQ)
    V = link_velocities(model, S, qd)
    inert = link_world_inertia(model, LP, LQ)
    M = crba(model, S, inert)
    C = rnea_bias(model, S, V, inert, qd, gravity)
    return np.linalg.solve(M, (tau - C)[..., None])[..., 0]


# ---------------------------------------------------------------- controllers

PD_JOINT_POS, PD_JOINT_DELTA_POS, PD_EE_DELTA_POSE = "pd_joint_pos", "pd_joint_delta_pos", "pd_ee_delta_pose"


def controller_targets(model, ctrl, q, action, control_freq=60):
    """SPEC.md:402-410 -> DriveTargets: (B, D) target positions and velocities.
    ctrl: mode, dofs (controlled dof indices), scale.  Uncontrolled dofs keep target = current q
    and target velocity 0 (with kp = kd = 0 they are undriven).

    pd_joint_pos        target = unnormalize(a) clamped; target velocity 0.
    pd_joint_delta_pos  target = clamp(q + a * scale); the delta is a motion over one control
                        period, so target velocity = (target - q) * control_freq.
    pd_ee_delta_pose twist = (a[0:3] * scale m in the world
                        frame, R_ee (a[3:6] * rot_scale) -- the axis-angle is given in the EE
                        frame and rotated to the world), at the ee link origin;
                        dq = J^T (J J^T + lam^2 I)^-1 twist over the controlled columns of the
                        geometric Jacobian; target = clamp(q + dq), velocity as for the joint
                        delta.
    base_forward_rotate velocity targets on the abstract base joints
                        (controlled dofs 0, 1, 2 = x, y, yaw): (a0 * scale cos yaw,
                        a0 * scale sin yaw, a1 * rot_scale) m/s, m/s, rad/s; position targets
                        stay at q (the base dofs carry kp = 0: a pure velocity servo)."""
    a = np.clip(np.asarray(action, np.float64), -1.0, 1.0)
    tgt = q.copy()
    tv = np.zeros_like(q)
    dofs = np.asarray(ctrl.dofs, dtype=np.int64)
    lo, hi = model.lower[dofs], model.upper[dofs]
    if ctrl.mode == PD_JOINT_DELTA_POS:
        tgt[:, dofs] = np.clip(q[:, dofs] + a * ctrl.scale, lo, hi)
        tv[:, dofs] = (tgt[:, dofs] - q[:, dofs]) * float(control_freq)
    elif ctrl.mode == PD_JOINT_POS:
        span_ok = np.isfinite(lo) & np.isfinite(hi)
        un = np.where(span_ok, lo + (a + 1.0) * 0.5 * (hi - lo), a * ctrl.scale)
        tgt[:, dofs] = np.clip(un, lo, hi)
    elif ctrl.mode == PD_EE_DELTA_POSE:
        LP, LQ = forward_kinematics(model, q)
        S = motion_subspace(model, LP, LQ)
        J = geometric_jacobian(model, S, ctrl.ee_link, LP[:, ctrl.ee_link])[:, :, dofs]
        w_ee = a[:, 3:6] * ctrl.rot_scale
        twist = np.concatenate([a[:, :3] * ctrl.scale, se3.qrot(LQ[:, ctrl.ee_link], w_ee)], -1)
        dq = ik_delta(J, twist, ctrl.lam)
        tgt[:, dofs] = np.clip(q[:, dofs] + dq, lo, hi)
        tv[:, dofs] = (tgt[:, dofs] - q[:, dofs]) * float(control_freq)
    elif ctrl.mode == "base_forward_rotate":
        a0, a1 = a[:, 0], a[:, 1]
        dx, dy, dyaw = dofs[0], dofs[1], dofs[2]
        yaw = q[:, dyaw]
        v = a0 * ctrl.scale
        tv[:, dx] = v * np.cos(yaw)
        tv[:, dy] = v * np.sin(yaw)
        tv[:, dyaw] = a1 * ctrl.rot_scale
    else:
        raise NotImplementedError(ctrl.mode)
    return tgt, tv


def control_step(model, st: State, drv: Drives, ctrl, action, cfg: SimConfig, want_contacts=False):
    drv.target, drv.target_vel = controller_targets(model, ctrl, st.q, action, cfg.control_freq)
    for _ in range(cfg.substeps):
        st = substep(model, st, drv, cfg, want_contacts)
    return st
