"""The oracle's articulated dynamics against the Euler-Lagrange equations (CPU only).

oracle/dynamics.py restates SPEC.md:328-336 with Featherstone's spatial algorithms (ABA, and
CRBA + RNEA as a cross-check, tests/test_oracle_dynamics.py).  This test pins them to first
principles with none of that code: the Lagrangian L = T - V of the chain is built from the link
poses alone (forward kinematics: the SPEC.md:256 KAT pins it), the link velocities by central
differences of those poses along qd, and the equations of motion
    d/dt (dL/dqd) - dL/dq = tau,   i.e.   M qdd = tau - Mdot qd + dT/dq - dV/dq
by finite differences of T and V (M_ij from the polarisation of the quadratic form T).
"""
import numpy as np
import pytest

from oracle import engine as E
from oracle import se3
from oracle.dynamics import forward_kinematics
from oracle.model import Model
from paper_2410_00425_b200.assets import load_urdf
from paper_2410_00425_b200.descriptors import ArticulationDesc, SceneDesc
from paper_2410_00425_b200 import fixtures as F

G = (0.0, 0.0, -9.81)
H = 1e-5


def _link_state(m, q):
    P, Q = forward_kinematics(m, q[None])
    com = P[0] + se3.qrot(Q[0], m.com)
    return com, Q[0]


def _T(m, q, qd):
    """Kinetic energy from pose differences: v_com and omega by central differences along qd."""
    c1, q1 = _link_state(m, q + H * qd)
    c0, q0 = _link_state(m, q - H * qd)
    v = (c1 - c0) / (2 * H)
    qdot = (q1 - q0) / (2 * H)
    _, Qm = _link_state(m, q)
    w = 2 * se3.qmul(qdot, se3.qconj(Qm))[:, 1:]  # world angular velocity
    R = se3.qmat(Qm)
    Iw = R @ m.inertia @ np.swapaxes(R, -1, -2)
    return 0.5 * float((m.mass * (v * v).sum(1)).sum() + np.einsum("li,lij,lj->", w, Iw, w))


def _V(m, q):
    com, _ = _link_state(m, q)
    return float(-(m.mass[:, None] * com * np.asarray(G)).sum())


def _M(m, q):
    """T = 1/2 qd' M qd is quadratic in qd: M_ii = 2 T(e_i), M_ij = T(e_i + e_j) - T(e_i) - T(e_j)."""
    D = len(q)
    e = np.eye(D)
    Ti = [_T(m, q, e[i]) for i in range(D)]
    return np.array([[2 * Ti[i] if i == j else _T(m, q, e[i] + e[j]) - Ti[i] - Ti[j] for j in range(D)]
                     for i in range(D)])


def _qdd_lagrange(m, q, qd, tau, h=1e-4):
    """M qdd = tau - Mdot qd + dT/dq - dV/dq, Mdot = sum_k dM/dq_k qd_k (central differences)."""
    D = len(q)
    e = np.eye(D)
    Mdot, dT, dV = np.zeros((D, D)), np.zeros(D), np.zeros(D)
    for k in range(D):
        Mdot += (_M(m, q + h * e[k]) - _M(m, q - h * e[k])) / (2 * h) * qd[k]
        dT[k] = (_T(m, q + h * e[k], qd) - _T(m, q - h * e[k], qd)) / (2 * h)
        dV[k] = (_V(m, q + h * e[k]) - _V(m, q - h * e[k])) / (2 * h)
    return np.linalg.solve(_M(m, q), tau - Mdot @ qd + dT - dV)


@pytest.mark.parametrize("urdf,dof", [(F.ARM3_URDF, 3), (F.make_chain_urdf(4), 4)])
def test_aba_matches_euler_lagrange(urdf, dof):
    m = Model(SceneDesc(articulations=(ArticulationDesc("a", load_urdf(urdf), (-0.2, 0.1, 0.3)),)))
    rng = np.random.default_rng(7)
    for _ in range(4):
        q, qd, tau = rng.uniform(-1.2, 1.2, dof), rng.normal(size=dof), rng.normal(size=dof)
        got = E.aba_qdd(m, q[None], qd[None], tau[None], G)[0]
        want = _qdd_lagrange(m, q, qd, tau)
        # (dropping the velocity terms misses by ~3 rad/s^2 here; the finite differences agree to ~1e-8 relative)
        assert np.abs(got - want).max() <= 1e-6 * max(1.0, np.abs(want).max()), (got, want)
