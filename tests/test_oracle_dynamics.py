"""Oracle pinning for the SPEC-only modules: the known-answer examples the reference states
for kinematics/dynamics/contacts (acceptance criteria SPEC.md:815-819).
CPU only; these are what make the oracle trustworthy where no reference code exists."""

import math

import numpy as np
import pytest

from oracle import engine as E
from oracle import se3
from oracle.contacts import detect_contacts, shape_world_poses
from oracle.dynamics import (forward_kinematics, geometric_jacobian, ik_delta, link_velocities,
                             motion_subspace)
from oracle.model import Model
from paper_2410_00425_b200 import fixtures as F
from paper_2410_00425_b200.assets import load_urdf
from paper_2410_00425_b200.descriptors import GROUND, ActorDesc, ArticulationDesc, SceneDesc, StaticDesc

G = (0.0, 0.0, -9.81)


def state_for(model, B, q=None, ap=None, aq=None):
    q = np.zeros((B, model.D)) if q is None else np.asarray(q, float).reshape(B, model.D)
    ap = np.zeros((B, model.A, 3)) if ap is None else np.asarray(ap, float).reshape(B, model.A, 3)
    aq = np.tile([1.0, 0, 0, 0], (B, model.A, 1)) if aq is None else np.asarray(aq, float).reshape(B, model.A, 4)
    return E.State(q, np.zeros_like(q), ap, aq, np.zeros((B, model.A, 3)), np.zeros((B, model.A, 3)),
                   np.zeros(B, np.uint8))


def no_drives(model, B):
    z = np.zeros(model.D)
    return E.Drives(z, z, np.full(model.D, np.inf), np.zeros((B, model.D)))


def run(model, st, n, cfg=None, drv=None):
    cfg = cfg or E.SimConfig()
    drv = drv or no_drives(model, st.q.shape[0])
    for _ in range(n):
        if drv.kp.any() is False:
            drv.target = st.q.copy()
        st = E.substep(model, st, drv, cfg)
    return st


def test_free_fall():
    m = Model(SceneDesc(actors=(ActorDesc("ball", "sphere", (0.1,)),)))
    st = run(m, state_for(m, 1), 120)
    assert abs(st.ap[0, 0, 2] - (-4.905)) <= 0.05
    assert st.av[0, 0, 2] == pytest.approx(-9.81, abs=1e-9)  # momentum: exact linear update


def test_fk_2r_and_arm3_zero_config():
    m = Model(SceneDesc(articulations=(ArticulationDesc("r", load_urdf(F.PLANAR_2R_URDF)),)))
    P, _ = forward_kinematics(m, np.array([[math.pi / 2, math.pi / 2]]))
    assert np.abs(P[0, 3] - [-1.0, 1.0, 0.0]).max() < 1e-9
    a = Model(SceneDesc(articulations=(ArticulationDesc("a", load_urdf(F.ARM3_URDF)),)))
    P, _ = forward_kinematics(a, np.zeros((1, 3)))
    assert np.abs(P[0, 3] - [0.4, 0, 0]).max() < 1e-12 and np.abs(P[0, 4] - [0.8, 0, 0]).max() < 1e-12


def test_fk_equals_compose_chain():
    tpl = load_urdf(F.make_chain_urdf(5))
    m = Model(SceneDesc(articulations=(ArticulationDesc("c", tpl, (0.1, -0.2, 0.3),
                                                        tuple(se3.qnorm(np.array([1.0, .2, .1, .3])))),)))
    rng = np.random.default_rng(0)
    q = rng.uniform(-1, 1, (4, 5))
    P, Q = forward_kinematics(m, q)
    p, qq = np.tile(m.org_p[0], (4, 1)), np.tile(m.org_q[0], (4, 1))
    for l in range(1, m.L):
        p, qq = se3.compose(p, qq, np.tile(m.org_p[l], (4, 1)), np.tile(m.org_q[l], (4, 1)))
        h = 0.5 * q[:, l - 1]
        mq = np.stack([np.cos(h), *(m.axis[l][k] * np.sin(h) for k in range(3))], -1)
        p, qq = se3.compose(p, qq, np.zeros((4, 3)), mq)
    assert np.abs(P[:, -1] - p).max() < 1e-12 and np.abs(Q[:, -1] - qq).max() < 1e-12


def test_jacobian_fd_and_dls():
    tpl = load_urdf(F.make_chain_urdf(4))
    m = Model(SceneDesc(articulations=(ArticulationDesc("c", tpl),)))
    rng = np.random.default_rng(1)
    q = rng.uniform(-1, 1, (50, 4))
    P, Q = forward_kinematics(m, q)
    S = motion_subspace(m, P, Q)
    J = geometric_jacobian(m, S, m.L - 1, P[:, -1])
    h = 1e-6
    for d in range(4):
        dq = np.zeros(4)
        dq[d] = h
        Pp, _ = forward_kinematics(m, q + dq)
        Pm, _ = forward_kinematics(m, q - dq)
        fd = (Pp[:, -1] - Pm[:, -1]) / (2 * h)
        assert np.abs(fd - J[:, :3, d]).max() < 1e-5
    # 2R zero config column 1 linear part = (0, 2, 0)
    r = Model(SceneDesc(articulations=(ArticulationDesc("r", load_urdf(F.PLANAR_2R_URDF)),)))
    P, Q = forward_kinematics(r, np.zeros((1, 2)))
    J = geometric_jacobian(r, motion_subspace(r, P, Q), 3, P[:, 3])
    assert np.abs(J[0, :3, 0] - [0, 2, 0]).max() < 1e-12
    # DLS == dense normal-equation solve and zero twist -> zero dq
    Jr = rng.normal(size=(20, 6, 4))
    tw = rng.normal(size=(20, 6))
    want = np.einsum("bji,bj->bi", Jr, np.linalg.solve(
        np.einsum("bij,bkj->bik", Jr, Jr) + 0.0025 * np.eye(6), tw[..., None])[..., 0])
    assert np.abs(ik_delta(Jr, tw) - want).max() < 1e-9
    assert np.abs(ik_delta(Jr, np.zeros_like(tw))).max() == 0.0


def test_pendulum_analytic_qacc():
    m = Model(SceneDesc(articulations=(ArticulationDesc("p", load_urdf(F.PENDULUM_URDF)),)))
    q = np.linspace(-3, 3, 13)[:, None]
    qdd = E.aba_qdd(m, q, np.zeros_like(q), np.zeros_like(q), G)
    # rotation about +y by q moves the bob (0,0,-1) to (-sin q, 0, -cos q): qdd = -(g/l) sin q
    assert np.abs(qdd[:, 0] - (-9.81 * np.sin(q[:, 0]))).max() < 1e-10


def test_aba_matches_crba_rnea_random_chains():
    rng = np.random.default_rng(2)
    for dof in (1, 2, 3, 4, 5):
        m = Model(SceneDesc(articulations=(ArticulationDesc("c", load_urdf(F.make_chain_urdf(dof))),)))
        B = 200
        q, qd, tau = rng.uniform(-1, 1, (B, dof)), rng.normal(size=(B, dof)), rng.normal(size=(B, dof))
        a = E.aba_qdd(m, q, qd, tau, G)
        b = E.crba_rnea_qdd(m, q, qd, tau, G)
        assert np.abs(a - b).max() < 1e-8
    # zero gravity / torque / velocity -> zero qdd
    z = np.zeros((3, 5))
    assert np.abs(E.aba_qdd(m, rng.uniform(-1, 1, (3, 5)), z, z, (0, 0, 0))).max() < 1e-12


def test_arm3_aba_matches_crba_rnea():
    m = Model(SceneDesc(articulations=(ArticulationDesc("a", load_urdf(F.ARM3_URDF), (-0.5, 0, 0.3)),)))
    rng = np.random.default_rng(3)
    q, qd, tau = rng.uniform(-1, 1, (100, 3)), rng.normal(size=(100, 3)), rng.normal(size=(100, 3))
    assert np.abs(E.aba_qdd(m, q, qd, tau, G) - E.crba_rnea_qdd(m, q, qd, tau, G)).max() < 1e-8


def test_pendulum_energy():
    m = Model(SceneDesc(articulations=(ArticulationDesc("p", load_urdf(F.LONG_PENDULUM_URDF)),)))
    st = state_for(m, 1, q=[[math.pi / 2]])
    l = 2.0
    energies = []
    for _ in range(1200):
        st = run(m, st, 1)
        th, w = st.q[0, 0], st.qd[0, 0]
        energies.append(0.5 * l * l * w * w + 9.81 * (-l * math.cos(th)))
    e0 = 0.0  # starts at rest at horizontal: E = 0
    amp = (max(energies) - min(energies)) / (9.81 * l)
    assert amp < 0.02, amp
    assert abs(np.mean(energies) - e0) < 0.02 * 9.81 * l


def contacts_of(desc, ap, aq=None):
    m = Model(desc)
    st = state_for(m, 1, ap=ap, aq=aq)
    P, Q = forward_kinematics(m, st.q)
    SP, SQ = shape_world_poses(m, P, Q, st.ap, st.aq)
    slots, unsup = detect_contacts(m, SP, SQ, 5e-4)
    return [(p[0], n[0], d[0]) for (_, p, n, d, v) in slots if v[0]], unsup


def test_contact_kats():
    c, _ = contacts_of(SceneDesc(actors=(ActorDesc("s", "sphere", (0.1,)),), statics=(GROUND,)), [[0, 0, 0.05]])
    assert len(c) == 1 and abs(c[0][2] - 0.05) < 1e-12 and np.allclose(c[0][1], [0, 0, 1])
    c, _ = contacts_of(SceneDesc(actors=(ActorDesc("b", "box", (0.5, 0.5, 0.5)),), statics=(GROUND,)), [[0, 0, 0.5]])
    assert len(c) == 4 and all(abs(d) < 1e-12 for (_, _, d) in c)
    c, _ = contacts_of(SceneDesc(actors=(ActorDesc("a", "sphere", (0.1,)), ActorDesc("b", "sphere", (0.1,)))),
                       [[0, 0, 0], [0.15, 0, 0]])
    assert len(c) == 1 and abs(c[0][2] - 0.05) < 1e-12 and np.allclose(c[0][1], [-1, 0, 0])


def test_resting_and_settling_sphere():
    desc = SceneDesc(actors=(ActorDesc("s", "sphere", (0.1,)),), statics=(GROUND,))
    m = Model(desc)
    st = run(m, state_for(m, 1, ap=[[0, 0, 0.1]]), 5)
    assert st.av[0, 0, 2] >= -1e-6
    st = run(m, state_for(m, 1, ap=[[0, 0, 0.5]]), 240)
    assert abs(st.ap[0, 0, 2] - 0.1) < 5e-4 + 1e-3


def test_box_on_incline_static_friction():
    ang = math.radians(20)  # tan(20 deg) = 0.36 < mu = 1: must not slide
    plane_q = (math.cos(ang / 2), math.sin(ang / 2), 0.0, 0.0)
    desc = SceneDesc(actors=(ActorDesc("b", "box", (0.05, 0.05, 0.05)),),
                     statics=(StaticDesc("incline", "plane", (), (0, 0, 0), plane_q),))
    m = Model(desc)
    n = se3.qrot(np.array(plane_q), np.array([0, 0, 1.0]))
    st = state_for(m, 1, ap=[0.05 * n], aq=[plane_q])
    st = run(m, st, 60)
    tang = st.av[0, 0] - np.dot(st.av[0, 0], n) * n
    st2 = run(m, st, 120)
    assert np.linalg.norm(st2.av[0, 0] - np.dot(st2.av[0, 0], n) * n) < 1e-3
    assert np.linalg.norm(st2.ap[0, 0] - st.ap[0, 0]) < 2e-3
    assert np.linalg.norm(tang) < 1e-2


def test_cube_rests_on_plane():
    desc = SceneDesc(actors=(ActorDesc("cube", "box", (0.02, 0.02, 0.02)),), statics=(GROUND,))
    m = Model(desc)
    st = run(m, state_for(m, 1, ap=[[0, 0, 0.02]]), 240)
    assert abs(st.ap[0, 0, 2] - 0.02) < 1.5e-3
    # sequential (Gauss-Seidel) box friction over 4 corners creeps slightly; bound it
    assert np.abs(st.ap[0, 0, :2]).max() < 1e-3
    assert np.linalg.norm(st.av[0, 0]) < 1e-2 and np.linalg.norm(st.aw[0, 0]) < 0.5


def test_free_body_momentum_conservation():
    """a free rigid body with no forces conserves linear momentum exactly and angular
    momentum within 1e-6 per second -- here an asymmetric brick tumbling fast in zero gravity
    (the gyroscopic case), over 2 s at 120 Hz (A-8: momentum transported to the new orientation)."""
    from oracle.model import Model
    from paper_2410_00425_b200.descriptors import ActorDesc, SceneDesc

    desc = SceneDesc((), (ActorDesc("brick", "box", (0.05, 0.02, 0.01), 1000.0, (0.5, 0.5, 0.5, 1.0)),), ())
    m = Model(desc)
    B = 8
    rng = np.random.default_rng(0)
    aq = se3.qnorm(rng.normal(size=(B, 1, 4)))
    st = E.State(np.zeros((B, 0)), np.zeros((B, 0)), np.zeros((B, 1, 3)), aq, rng.normal(size=(B, 1, 3)),
                 rng.normal(size=(B, 1, 3)) * 5.0, np.zeros(B, np.uint8))
    drv = E.Drives(np.zeros(0), np.zeros(0), np.zeros(0), np.zeros((B, 0)), np.zeros((B, 0)))
    cfg = E.SimConfig(gravity=(0.0, 0.0, 0.0))

    def ang_mom(s):
        Iw, _ = E.actor_world_inertia(m, s.aq)
        return np.einsum("baij,baj->bai", Iw, s.aw)

    L0, p0 = ang_mom(st), st.av.copy()
    for _ in range(240):
        st = E.substep(m, st, drv, cfg)
    rel = np.linalg.norm(ang_mom(st) - L0, axis=-1) / np.linalg.norm(L0, axis=-1)
    assert rel.max() < 2e-6, rel.max()            # <= 1e-6 per second over 2 s
    assert np.array_equal(st.av, p0)               # linear momentum exactly
    assert np.abs(np.linalg.norm(st.aq, axis=-1) - 1.0).max() < 1e-12
