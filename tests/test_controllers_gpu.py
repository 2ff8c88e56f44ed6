"""Controller semantics and the scene invariants of the SPEC on the GPU product, vs the oracle.

  * pd_joint_pos in the fused step kernel: targets and stepped state == oracle.
  * Hold property: pd_joint_delta_pos, zero actions, gravity-compensated fixture
    (ARM3 alone, gravity off): qpos drift < 1e-3 rad over 100 steps; device == oracle.
  * SPEC.md:409 KAT on a reachable (6-DOF) arm: +x twist of 0.01 m per step, after 10 steps
    the EE x has advanced >= 0.05 m and within +-30% of 0.1 m, with the SPEC drive model
    (target velocity, gains per unit inertia); device == oracle step by step.
  * Heterogeneity equivalence (acceptance criterion SPEC.md:818): a batch
    of 8 OpenCabinet envs with 2-6 cabinet DOF (5-9 total) stepped 500 times equals, env by
    env, the same env simulated ALONE (its own 1-env batch: D_max = its DOF, a different
    kernel width) with the same seed and substeps, within 1e-10.
  * Free-body momentum: an asymmetric brick tumbling in zero gravity keeps its
    angular momentum to 1e-6 per second and its linear momentum exactly; device == oracle.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _state(env):
    s = env.scene
    return s.qpos.cpu().numpy(), s.qvel.cpu().numpy()


def test_pd_joint_pos_in_kernel_parity(cuda):
    from oracle import engine as E
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.tasks import make_task, pickcube_scene

    N = 16
    env = make_task("PickCube", N, seed=3, overrides={"control_mode": "pd_joint_pos", "action_scale": 1.0})
    orc = PickCubeOracle(env.spec, pickcube_scene(env.spec), N, 3)
    rng = np.random.default_rng(4)
    for t in range(20):
        s = env.scene
        ap, av = s.actor_pose.cpu().numpy(), s.actor_vel.cpu().numpy()
        orc.load({"q": s.qpos.cpu().numpy(), "qd": s.qvel.cpu().numpy(), "ap": ap[:, :, :3], "aq": ap[:, :, 3:],
                  "av": av[:, :, :3], "aw": av[:, :, 3:], "goal": s.goal.cpu().numpy(),
                  "elapsed": s.elapsed.cpu().numpy()})
        orc.reset_count[:] = s.reset_count.cpu().numpy().astype(np.uint64)
        a = rng.uniform(-1.2, 1.2, (N, 3)).astype(np.float32)  # out-of-range actions are clipped
        want_tgt, want_tv = E.controller_targets(orc.model, orc.ctrl, orc.st.q, a, 60)
        assert (want_tv == 0).all()
        r = env.step(torch.as_tensor(a, device=env.device))
        _, o_rew, o_term, o_trunc, _, final = orc.step(a)
        done = (o_term | o_trunc)
        tg = s.target.cpu().numpy()
        assert np.abs(tg[~done] - want_tgt[~done]).max() <= 1e-12, t
        assert np.array_equal(r.terminated.cpu().numpy().astype(bool), o_term), t
        snap = orc.snapshot()
        q, qd = _state(env)
        assert np.abs(q - snap["q"]).max() <= 1e-9, t
        assert np.abs(qd - snap["qd"]).max() <= 1e-9, t


def _arm_env(urdf, mode, n, gravity, scale, q0):
    from paper_2410_00425_b200 import cabi
    from paper_2410_00425_b200.assets import load_urdf
    from paper_2410_00425_b200.descriptors import ArticulationDesc, ControlSpec, SceneDesc
    from paper_2410_00425_b200.envs import Env, SimConfig
    from paper_2410_00425_b200.scene import build_batch

    desc = SceneDesc((ArticulationDesc("arm", load_urdf(urdf), (-0.5, 0.0, 0.25)),), (), ())
    ctl = ControlSpec(mode, "arm", action_scale=scale)
    scene = build_batch([desc] * n, 0, ctl)
    ee = scene.models[0].link_names.index("arm/ee")
    env = Env(scene, cabi.TASK_NONE, [0.0] * 9, ee, 10 ** 6, 0, sim=SimConfig(gravity=gravity), auto_reset=False,
              name="Arm")
    env.reset()
    env.scene.qpos[:, :len(q0[0])] = torch.as_tensor(q0, device=env.device)
    env.scene.forward_kinematics()
    return env, desc, ctl


def _oracle_for(desc, ctl, mode, scale, gravity):
    from oracle import engine as E
    from oracle.model import Model

    m = Model(desc)
    D = m.D
    drv = E.Drives(np.full(D, ctl.kp), np.full(D, ctl.kd), np.full(D, ctl.force_limit), None)
    ctrl = type("C", (), {"mode": mode, "dofs": list(range(D)), "scale": scale, "rot_scale": ctl.action_scale_rot,
                          "lam": ctl.ik_lambda, "ee_link": m.link_names.index("arm/ee")})()
    return m, drv, ctrl, E.SimConfig(gravity=gravity)


def test_hold_property_gpu(cuda):
    from oracle import engine as E
    from paper_2410_00425_b200.fixtures import ARM3_URDF

    B = 8
    rng = np.random.default_rng(1)
    q0 = np.array([0.0, -0.3, 1.2]) + rng.uniform(-0.5, 0.5, (B, 3))
    qd0 = rng.uniform(-0.02, 0.02, (B, 3))
    g0 = (0.0, 0.0, 0.0)
    env, desc, ctl = _arm_env(ARM3_URDF, "pd_joint_delta_pos", B, g0, 0.1, q0)
    env.scene.qvel[:, :3] = torch.as_tensor(qd0, device=env.device)
    m, drv, ctrl, cfg = _oracle_for(desc, ctl, "pd_joint_delta_pos", 0.1, g0)
    st = E.State(q0.copy(), qd0.copy(), np.zeros((B, 0, 3)), np.zeros((B, 0, 4)), np.zeros((B, 0, 3)),
                 np.zeros((B, 0, 3)), np.zeros(B, np.uint8))
    zero = torch.zeros((B, 3), device=env.device)
    for t in range(100):
        env.step(zero)
        st = E.control_step(m, st, drv, ctrl, np.zeros((B, 3)), cfg)
        q, qd = _state(env)
        assert np.abs(q - q0).max() < 1e-3, t
        assert np.abs(q - st.q).max() <= 1e-9 and np.abs(qd - st.qd).max() <= 1e-9, t


def test_ee_delta_pose_kat_reachable_arm_gpu(cuda):
    from oracle import engine as E
    from oracle.dynamics import forward_kinematics
    from paper_2410_00425_b200.fixtures import ARM6_URDF

    B = 4
    q0 = np.tile([0.0, -0.3, 1.2, 0.0, -0.6, 0.0], (B, 1))
    g = (0.0, 0.0, -9.81)
    env, desc, ctl = _arm_env(ARM6_URDF, "pd_ee_delta_pose", B, g, 0.01, q0)
    assert env.action_dim == 6
    m, drv, ctrl, cfg = _oracle_for(desc, ctl, "pd_ee_delta_pose", 0.01, g)
    st = E.State(q0.copy(), np.zeros((B, 6)), np.zeros((B, 0, 3)), np.zeros((B, 0, 4)), np.zeros((B, 0, 3)),
                 np.zeros((B, 0, 3)), np.zeros(B, np.uint8))
    a = np.zeros((B, 6), np.float32)
    a[:, 0] = 1.0
    a[1, 3:] = (0.0, 0.0, 0.3)   # the other envs also rotate (EE-frame axis-angle)
    a[2, 3:] = (0.4, -0.2, 0.0)
    ee = ctrl.ee_link
    p0 = env.scene.link_pose.cpu().numpy()[:, ee, :3].copy()
    for t in range(10):
        env.step(torch.as_tensor(a, device=env.device))
        st = E.control_step(m, st, drv, ctrl, a, cfg)
        q, qd = _state(env)
        assert np.abs(q - st.q).max() <= 1e-9 and np.abs(qd - st.qd).max() <= 1e-9, t
    p1 = env.scene.link_pose.cpu().numpy()[:, ee, :3]
    dx = p1[:, 0] - p0[:, 0]
    assert dx[0] >= 0.05 and abs(dx[0] - 0.1) <= 0.03, dx  # SPEC.md:409 (pure +x twist)
    LP, _ = forward_kinematics(m, st.q)
    assert np.abs(LP[:, ee] - p1).max() <= 1e-9


def test_heterogeneity_equivalence_500_steps(cuda):
    from paper_2410_00425_b200 import cabi
    from paper_2410_00425_b200.envs import Env
    from paper_2410_00425_b200.scene import SceneBatch
    from paper_2410_00425_b200.tasks import make_task

    N, SEED, STEPS = 8, 2, 500
    batch = make_task("OpenCabinet", N, seed=SEED)
    dofs = [batch.scene.models[m].D for m in batch.scene.model_index]
    assert len(set(dofs)) >= 3, dofs
    spec = batch.spec
    solos = []
    for e in range(N):
        sc = SceneBatch([batch.descs[e]], spec.control(), batch.device, env_offset=e)
        ee = sc.models[0].link_names.index(f"arm/{spec.ee_link}")
        solo = Env(sc, cabi.TASK_OPENCHAIN, spec.task_f(), ee, spec.max_steps, SEED, name="OpenCabinet")
        solo.reset()
        assert solo.scene.D_max == dofs[e]
        solos.append(solo)
    a = torch.empty((N, 3), dtype=torch.float32, device=batch.device)
    from paper_2410_00425_b200 import _native as nat

    worst = 0.0
    resets = 0
    for t in range(STEPS):
        nat.call("bs_random_actions", SEED, t, 0, N, 3, a.data_ptr(), nat.stream_handle())
        r = batch.step(a)
        resets += int((r.terminated | r.truncated).sum())
        for e in range(N):
            solos[e].step(a[e:e + 1].clone())
        if t % 25 == 24 or t == STEPS - 1:
            q, qd = _state(batch)
            for e in range(N):
                d = dofs[e]
                qs, qds = _state(solos[e])
                err = max(np.abs(q[e, :d] - qs[0, :d]).max(), np.abs(qd[e, :d] - qds[0, :d]).max())
                worst = max(worst, err)
                assert err <= 1e-10, (t, e, err)
                assert (q[e, d:] == 0).all() and (qd[e, d:] == 0).all()  # padding stays zero
    print(f"heterogeneity equivalence: max |batch - solo| = {worst:.3e} over {STEPS} steps, {resets} resets")


def test_free_body_momentum_gpu(cuda):
    """SPEC.md:358 on the device: an asymmetric brick tumbling in zero gravity (no contacts)
    conserves angular momentum to <= 1e-6 per second and linear momentum exactly; state ==
    oracle within 1e-9 (A-8 momentum transport)."""
    from oracle import engine as E
    from oracle import se3
    from oracle.model import Model
    from paper_2410_00425_b200 import cabi
    from paper_2410_00425_b200.descriptors import ActorDesc, ControlSpec, SceneDesc
    from paper_2410_00425_b200.envs import Env, SimConfig
    from paper_2410_00425_b200.scene import build_batch

    desc = SceneDesc((), (ActorDesc("brick", "box", (0.05, 0.02, 0.01), 1000.0, (0.5, 0.5, 0.5, 1.0)),), ())
    B = 8
    scene = build_batch([desc] * B, 0, ControlSpec())
    env = Env(scene, cabi.TASK_NONE, [0.0] * 9, -1, 10 ** 6, 0, sim=SimConfig(gravity=(0.0, 0.0, 0.0)),
              auto_reset=False, name="Brick")
    env.reset()
    rng = np.random.default_rng(0)
    aq = se3.qnorm(rng.normal(size=(B, 1, 4)))
    av, aw = rng.normal(size=(B, 1, 3)), rng.normal(size=(B, 1, 3)) * 5.0
    pose = np.concatenate([np.zeros((B, 1, 3)), aq], -1)
    env.scene.actor_pose.copy_(torch.as_tensor(pose, device=env.device))
    env.scene.actor_vel.copy_(torch.as_tensor(np.concatenate([av, aw], -1), device=env.device))
    m = Model(desc)
    st = E.State(np.zeros((B, 0)), np.zeros((B, 0)), np.zeros((B, 1, 3)), aq.copy(), av.copy(), aw.copy(),
                 np.zeros(B, np.uint8))
    drv = E.Drives(np.zeros(0), np.zeros(0), np.zeros(0), np.zeros((B, 0)), np.zeros((B, 0)))
    cfg = E.SimConfig(gravity=(0.0, 0.0, 0.0))
    I_b = np.asarray(m.actor_inertia[0])

    def ang_mom(q, w):
        R = se3.qmat(q)
        return np.einsum("bij,j,bkj,bk->bi", R, I_b, R, w)

    L0 = ang_mom(aq[:, 0], aw[:, 0])
    act = torch.zeros((B, 0), device=env.device)
    for t in range(60):  # 1 s of 120 Hz substeps
        env.step(act)
        st = E.control_step(m, st, drv, type("C", (), {"mode": "pd_joint_pos", "dofs": [], "scale": 1.0})(),
                            np.zeros((B, 0)), cfg)
    p = env.scene.actor_pose.cpu().numpy()[:, 0]
    v = env.scene.actor_vel.cpu().numpy()[:, 0]
    assert np.abs(p[:, 3:] - st.aq[:, 0]).max() <= 1e-9 and np.abs(v[:, 3:] - st.aw[:, 0]).max() <= 1e-9
    rel = np.linalg.norm(ang_mom(p[:, 3:], v[:, 3:]) - L0, axis=-1) / np.linalg.norm(L0, axis=-1)
    assert rel.max() <= 1e-6, rel.max()
    assert np.array_equal(v[:, :3], av[:, 0])
