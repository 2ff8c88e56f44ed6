"""GPU fused step vs the CPU oracle on the PickCube-style task (config C1: 16 envs, 200
steps, fp64).

Bars (BASELINE north star): integer outputs bit-exact (contact pair lists, success/fail/
terminated/truncated flags, unsupported-pair counters, env indexing, random actions);
float state within a stated tolerance:
  * one-step parity from an identical state: |dx| <= 1e-9 (abs, m / rad / m/s);
  * 200-step free-running trajectory: relative 1e-4 on body/articulation state.
"""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, STEPS, SEED = 16, 200, 7


@pytest.fixture(scope="module")
def pair(cuda):
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.tasks import make_task, pickcube_scene

    env = make_task("PickCube", N, seed=SEED)
    orc = PickCubeOracle(env.spec, pickcube_scene(env.spec), N, SEED)
    return env, orc


def gpu_snapshot(env):
    s = env.scene
    ap = s.actor_pose.cpu().numpy()
    av = s.actor_vel.cpu().numpy()
    return {"q": s.qpos.cpu().numpy()[:, :3], "qd": s.qvel.cpu().numpy()[:, :3], "ap": ap[:, :, :3],
            "aq": ap[:, :, 3:], "av": av[:, :, :3], "aw": av[:, :, 3:], "goal": s.goal.cpu().numpy(),
            "elapsed": s.elapsed.cpu().numpy()}


def compare(a, b, atol, rtol=0.0, what=""):
    for k in ("q", "qd", "ap", "aq", "av", "aw", "goal"):
        x, y = np.asarray(a[k], np.float64), np.asarray(b[k], np.float64)
        err = np.abs(x - y)
        lim = atol + rtol * np.abs(y)
        assert (err <= lim).all(), f"{what} {k}: max err {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"


def actions(env, step):
    from oracle.philox import action_uniforms

    got = torch.empty((N, env.action_dim), dtype=torch.float32, device=env.device)
    from paper_2410_00425_b200 import _native as nat

    nat.call("bs_random_actions", SEED, step, 0, N, env.action_dim, got.data_ptr(), nat.stream_handle())
    want = action_uniforms(SEED, step, np.arange(N), env.action_dim)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32)), "Philox actions differ"
    return got, want


def test_reset_matches_oracle(pair):
    env, orc = pair
    env.reset(seed=SEED)
    orc.reset_count[:] = 0
    orc.reset()
    g = gpu_snapshot(env)
    o = orc.snapshot()
    assert np.array_equal(g["q"], o["q"]), "qpos reset is exact arithmetic"
    assert np.array_equal(g["ap"], o["ap"]) and np.array_equal(g["goal"], o["goal"])
    compare(g, o, atol=1e-15, what="reset")
    obs = env.state_obs.cpu().numpy()
    oo = orc.obs()
    assert np.abs(obs - oo).max() <= 1e-6


def test_one_step_parity_and_integer_outputs(pair):
    env, orc = pair
    env.reset(seed=SEED)
    orc.reset_count[:] = 0
    orc.reset()
    n_contacts = 0
    for t in range(60):
        orc.load(gpu_snapshot(env))
        orc.reset_count[:] = env.scene.reset_count.cpu().numpy().astype(np.uint64)
        a_gpu, a_np = actions(env, t)
        r = env.step(a_gpu)
        _, o_rew, o_term, o_trunc, o_info, final = orc.step(a_np, want_contacts=True)
        # integer outputs: bit-exact
        assert np.array_equal(r.info["unsupported_pairs"].cpu().numpy(), o_info["unsupported_pairs"])
        assert np.array_equal(r.terminated.cpu().numpy().astype(bool), o_term)
        assert np.array_equal(r.truncated.cpu().numpy().astype(bool), o_trunc)
        assert np.array_equal(r.info["success"].cpu().numpy().astype(bool), o_info["success"])
        cnt, pairs, geom = (x.cpu().numpy() for x in env.contacts())
        for e in range(N):
            want = [(i, j) for (i, j, P, n, d, v) in o_info["contacts"] if v[e]]
            got = [tuple(pairs[e, c]) for c in range(cnt[e])]
            assert got == want, f"step {t} env {e}: contact pairs {got} != {want}"
            wg = np.array([np.concatenate([P[e], n[e], [d[e]]]) for (i, j, P, n, d, v) in o_info["contacts"] if v[e]])
            if len(wg):
                assert np.abs(geom[e, :cnt[e]] - wg).max() < 1e-9
            n_contacts += cnt[e]
        assert np.abs(r.reward.cpu().numpy() - o_rew).max() < 1e-5
        # float state after the step (post auto-reset): tight tolerance
        compare(gpu_snapshot(env), orc.snapshot(), atol=1e-9, what=f"step {t}")
    assert n_contacts > 0, "the trajectory never touched anything"


def test_trajectory_parity_200_steps(pair):
    env, orc = pair
    env.reset(seed=SEED)
    orc.reset_count[:] = 0
    orc.reset()
    worst = 0.0
    for t in range(STEPS):
        a_gpu, a_np = actions(env, t)
        r = env.step(a_gpu)
        _, o_rew, o_term, o_trunc, o_info, _ = orc.step(a_np)
        assert np.array_equal(r.terminated.cpu().numpy().astype(bool), o_term), f"step {t}"
        assert np.array_equal(r.truncated.cpu().numpy().astype(bool), o_trunc), f"step {t}"
        g, o = gpu_snapshot(env), orc.snapshot()
        compare(g, o, atol=1e-7, rtol=1e-4, what=f"trajectory step {t}")
        worst = max(worst, max(np.abs(np.asarray(g[k]) - np.asarray(o[k])).max() for k in ("q", "ap")))
    print(f"max |dx| over {STEPS} steps: {worst:.3e}")


def test_determinism_and_snapshot(pair):
    env, _ = pair
    env.reset(seed=3)
    snap = env.scene.get_state()
    for t in range(10):
        env.step_random(t)
    a = env.scene.get_state()
    env.scene.set_state(snap)
    for t in range(10):
        env.step_random(t)
    b = env.scene.get_state()
    for k in env.scene.STATE_FIELDS:
        assert torch.equal(a[k], b[k]), k
    # partial set_state: env 1 untouched bitwise
    mask = torch.zeros(N, dtype=torch.uint8)
    mask[0] = 1
    before = env.scene.get_state()
    env.scene.set_state(snap, env_mask=mask)
    after = env.scene.get_state()
    for k in env.scene.STATE_FIELDS:
        assert torch.equal(after[k][1:], before[k][1:]), k
        assert torch.equal(after[k][0], snap[k][0]), k


def test_cross_env_independence(pair):
    env, _ = pair
    env.reset(seed=11)
    snap = env.scene.get_state()
    for t in range(20):
        env.step_random(t)
    ref = env.scene.get_state()
    env.scene.set_state(snap)
    env.scene.qvel[5, 1] += 0.5  # perturb env 5 only
    for t in range(20):
        env.step_random(t)
    got = env.scene.get_state()
    for k in ("qpos", "qvel", "actor_pose", "actor_vel"):
        keep = torch.ones(N, dtype=torch.bool)
        keep[5] = False
        assert torch.equal(got[k][keep], ref[k][keep]), k
    # the perturbed env itself moved differently (its arm; the cube may be untouched)
    assert not torch.equal(got["qpos"][5], ref["qpos"][5])


def test_shard_equivalence(cuda):
    """Global env indices key the RNG: two shards == one batch, bitwise."""
    from paper_2410_00425_b200.tasks import make_task

    full = make_task("PickCube", 8, seed=5)
    lo = make_task("PickCube", 8, seed=5, shard=(0, 2))
    hi = make_task("PickCube", 8, seed=5, shard=(1, 2))
    for t in range(15):
        full.step_random(t)
        lo.step_random(t)
        hi.step_random(t)
    for k in ("qpos", "qvel", "actor_pose", "actor_vel", "goal"):
        cat = torch.cat([getattr(lo.scene, k), getattr(hi.scene, k)])
        assert torch.equal(cat, getattr(full.scene, k)), k


def test_graph_replay_matches_eager(cuda):
    from paper_2410_00425_b200.tasks import make_task

    a = make_task("PickCube", 64, seed=9)
    b = make_task("PickCube", 64, seed=9)
    b.capture_graph()
    for t in range(12):
        a.step_random(t)
        b.step_random(t)
    for k in ("qpos", "qvel", "actor_pose", "actor_vel", "elapsed"):
        assert torch.equal(getattr(a.scene, k), getattr(b.scene, k)), k


def test_nonfinite_action_raises(cuda):
    from paper_2410_00425_b200.errors import InputError
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickCube", 4, seed=0)
    a = torch.zeros((4, 3), device=env.device)
    a[2, 1] = float("nan")
    with pytest.raises(InputError):
        env.step(a)


def test_divergence_flags_and_freezes_only_that_env(cuda):
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickCube", 4, seed=0, auto_reset=False)
    env.scene.qvel[2, 0] = float("inf")
    before = env.scene.get_state()
    r = env.step(torch.zeros((4, 3), device=env.device))
    assert env.scene.diverged.cpu().tolist() == [0, 0, 1, 0]
    assert bool(r.info["fail"][2]) and bool(r.terminated[2])
    assert torch.equal(env.scene.qpos[2], before["qpos"][2])  # frozen
    assert torch.isfinite(env.scene.qpos[[0, 1, 3]]).all()


def test_ee_delta_pose_one_step_parity(cuda):
    """pd_ee_delta_pose (DLS IK) on the device vs the oracle: targets and
    the stepped state within 1e-9 from identical start states."""
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.tasks import make_task, pickcube_scene

    ov = {"control_mode": "pd_ee_delta_pose", "action_scale": 0.01}
    env = make_task("PickCube", 8, seed=13, overrides=ov)
    assert env.action_dim == 6
    orc = PickCubeOracle(env.spec, pickcube_scene(env.spec), 8, 13)
    rng = np.random.default_rng(0)
    for t in range(15):
        orc.load(gpu_snapshot(env))
        orc.reset_count[:] = env.scene.reset_count.cpu().numpy().astype(np.uint64)
        a = rng.uniform(-1, 1, (8, 6)).astype(np.float32)
        env.step(torch.as_tensor(a, device=env.device))
        orc.step(a)
        tg = env.scene.target.cpu().numpy()[:, :3]
        assert np.isfinite(tg).all()
        compare(gpu_snapshot(env), orc.snapshot(), atol=1e-9, what=f"ee step {t}")


def test_episode_metrics_match_oracle(cuda):
    """In-kernel EpisodeMetrics vs the oracle accumulator on short episodes:
    done masks, lengths and flags bit-exact; returns within 1e-6 relative."""
    from oracle.metrics import EpisodeAccumulator
    from oracle.philox import action_uniforms
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.metrics import EpisodeStats
    from paper_2410_00425_b200.tasks import make_task, pickcube_scene

    env = make_task("PickCube", N, seed=21, overrides={"max_steps": 4})
    orc = PickCubeOracle(env.spec, pickcube_scene(env.spec), N, 21)
    acc = EpisodeAccumulator(N)
    stats = EpisodeStats(env.device)
    episodes = 0
    for t in range(13):
        r = env.step_random(t)
        stats.update(r.info)
        _, o_rew, o_term, o_trunc, o_info, final = orc.step(action_uniforms(21, t, np.arange(N), 3))
        done, ret, length, flags = acc.update(o_rew, o_info["success"], o_info["fail"], o_term, o_trunc,
                                              final["elapsed"])
        ep = r.info["episode"]
        g_done = ep["done"].cpu().numpy().astype(bool)
        assert np.array_equal(g_done, done), t
        if done.any():
            assert np.array_equal(ep["length"].cpu().numpy()[done], length[done])
            assert np.array_equal(ep["flags"].cpu().numpy()[done], flags[done])
            g_ret = ep["return"].cpu().numpy()[done]
            assert np.abs(g_ret - ret[done]).max() <= 1e-6 * (1 + np.abs(ret[done]).max())
            episodes += int(done.sum())
    assert episodes >= 3 * N
    assert int(stats.sums[0]) == episodes


@pytest.mark.parametrize("task,obs_mode,over", [
    ("PickCube", "rgbd", None),
    ("PickCube", "rgb+depth+seg", None),
    ("PickCube", "pointcloud", None),
    ("PickHetero", "rgb+depth+seg", {"camera_res": 64}),  # two cameras in one group
])
def test_step_host_matches_device_step(cuda, task, obs_mode, over):
    """Env.step_host (one graph: step with zero-copy host actions and obs/reward/flags, render, D2H
    of the images and of the device-derived entries such as the pointcloud mask) == Env.step,
    every returned array bitwise, several steps in a row (auto-resets included)."""
    from paper_2410_00425_b200.envs import Env
    from paper_2410_00425_b200.tasks import make_task

    a = make_task(task, 8, seed=17, obs_mode=obs_mode, overrides=over)
    b = make_task(task, 8, seed=17, obs_mode=obs_mode, overrides=over)
    rng = np.random.default_rng(2)
    for t in range(6):
        act = rng.uniform(-1, 1, (8, a.action_dim)).astype(np.float32)
        ra = a.step(torch.as_tensor(act, device=a.device))
        hb = b.step_host(act)
        dev = {"reward": ra.reward, **{k: getattr(a, k) for k in ("terminated", "truncated", "success", "fail")}}
        dev.update(Env._flatten_obs(ra.obs))
        assert set(dev) == set(hb), (sorted(dev), sorted(hb))
        for k, v in dev.items():
            assert np.array_equal(v.cpu().numpy(), hb[k].numpy()), (t, k)
    h2d, d2h = b.host_io_bytes()
    assert h2d == 8 * a.action_dim * 4 and d2h > 8 * 64 * 64


def test_base_forward_rotate_matches_oracle(cuda):
    """base_forward_rotate: 2-D action (forward, rotate) -> VELOCITY
    targets of an abstract mobile base (m/s along the heading, rad/s); device == oracle within
    1e-9, and the base drives along its heading at the commanded speed."""
    import math

    from oracle import engine as E
    from oracle.model import Model
    from paper_2410_00425_b200 import cabi
    from paper_2410_00425_b200.assets import load_urdf
    from paper_2410_00425_b200.descriptors import GROUND, ArticulationDesc, ControlSpec, SceneDesc
    from paper_2410_00425_b200.envs import Env
    from paper_2410_00425_b200.fixtures import make_mobile_base_urdf
    from paper_2410_00425_b200.scene import build_batch

    desc = SceneDesc((ArticulationDesc("base", load_urdf(make_mobile_base_urdf())),), (), (GROUND,))
    ctl = ControlSpec("base_forward_rotate", "base", action_scale=0.5, action_scale_rot=1.0)
    scene = build_batch([desc] * 4, 0, ctl)
    env = Env(scene, cabi.TASK_NONE, [0.0] * 9, -1, 1000, 0, name="DriveBase")
    env.reset()
    assert env.action_dim == 2
    m = Model(desc)
    # the base joints are velocity servos: kp = 0, kd per unit inertia
    drv = E.Drives(np.zeros(3), np.full(3, ctl.kd), np.full(3, ctl.force_limit), np.zeros((4, 3)))
    ctrl = type("C", (), {"mode": "base_forward_rotate", "dofs": [0, 1, 2], "scale": 0.5, "rot_scale": 1.0})()
    rng = np.random.default_rng(5)
    for t in range(30):  # the 100 N force limit takes ~9 steps to reach 0.5 m/s
        q0, qd0 = env.scene.qpos.cpu().numpy(), env.scene.qvel.cpu().numpy()
        st = E.State(q0.copy(), qd0.copy(), np.zeros((4, 0, 3)), np.zeros((4, 0, 4)), np.zeros((4, 0, 3)),
                     np.zeros((4, 0, 3)), np.zeros(4, np.uint8))
        a = rng.uniform(-1, 1, (4, 2)).astype(np.float32)
        a[:, 0] = 1.0
        env.step(torch.as_tensor(a, device=env.device))
        st = E.control_step(m, st, drv, ctrl, a, E.SimConfig())
        assert np.abs(env.scene.qpos.cpu().numpy() - st.q).max() < 1e-9, t
    q = env.scene.qpos.cpu().numpy()
    qd = env.scene.qvel.cpu().numpy()
    assert (np.hypot(q[:, 0], q[:, 1]) > 0.15).all()  # moved forward along the heading
    speed = np.hypot(qd[:, 0], qd[:, 1])
    assert np.abs(speed - 0.5).max() < 0.05, speed  # tracking the 0.5 m/s velocity target


def test_generic_width_kernel_variant(cuda):
    """The PickCube scene normally runs the static-width kernel variant (D_max == 3, A_max == 1);
    rerun the parity tests of this module on the runtime-width variant (BS_STEP_GENERIC=1)."""
    import os
    import subprocess
    import sys

    if os.environ.get("BS_STEP_GENERIC"):
        pytest.skip("already running the generic variant")
    env = dict(os.environ, BS_STEP_GENERIC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__, "-k",
                        "one_step_parity or trajectory_parity or ee_delta or episode_metrics"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("lanes", [8, 16, 32])
def test_lane_count_variants(cuda, lanes):
    """bs_step picks 8, 16 or 32 lanes per env from the batch size (small batches get more lanes
    per env); force each variant (BS_STEP_G) and rerun the parity tests of this module and the
    cabinet (articulated-variant) tests on it."""
    import os
    import subprocess
    import sys

    if os.environ.get("BS_STEP_G") or os.environ.get("BS_STEP_GENERIC"):
        pytest.skip("already running a forced variant")
    env = dict(os.environ, BS_STEP_G=str(lanes))
    here = os.path.dirname(__file__)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__,
                        os.path.join(here, "test_cabinet_gpu.py"), "-k",
                        "one_step_parity or trajectory_parity or ee_delta or episode_metrics or cabinet"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_graph_recaptures_after_param_changes(cuda):
    """A captured graph bakes in BsSimParams: reset(seed=new) and eval_wrapper change them, so the
    next replay must re-capture -- graph and eager runs stay bitwise equal through both."""
    from paper_2410_00425_b200.metrics import eval_wrapper
    from paper_2410_00425_b200.tasks import make_task

    a = make_task("PickCube", 32, seed=9, overrides={"max_steps": 5})
    b = make_task("PickCube", 32, seed=9, overrides={"max_steps": 5})
    b.capture_graph()
    for seed in (9, 123):
        a.reset(seed=seed)
        b.reset(seed=seed)
        for t in range(12):  # crosses two auto-resets, which draw from the new seed's streams
            a.step_random(t)
            b.step_random(t)
        for k in ("qpos", "qvel", "actor_pose", "goal", "elapsed", "reset_count"):
            assert torch.equal(getattr(a.scene, k), getattr(b.scene, k)), (seed, k)
    eval_wrapper(a)
    eval_wrapper(b)
    for t in range(8):
        ra = a.step_random(t)
        rb = b.step_random(t)
        assert torch.equal(ra.terminated, rb.terminated) and not bool(rb.terminated.any())
    assert torch.equal(a.scene.elapsed, b.scene.elapsed) and int(b.scene.elapsed.max()) > 5  # no auto-reset


def test_host_graph_follows_eval_wrapper(cuda):
    from paper_2410_00425_b200.metrics import eval_wrapper
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickCube", 8, seed=2, overrides={"max_steps": 3})
    act = np.zeros((8, 3), np.float32)
    env.step_host(act)
    eval_wrapper(env)
    for _ in range(6):
        out = env.step_host(act)
        assert not out["terminated"].numpy().any()
    assert int(env.scene.elapsed.min()) == 7  # never auto-reset in eval mode


def test_capture_leaves_no_trace(cuda):
    """Capturing (and its warmup) restores the scene state AND the outputs: the obs returned by
    reset() still describes the current state afterwards."""
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickCube", 16, seed=4, obs_mode="rgbd")
    obs = env.reset(seed=4)
    st0 = {k: v.clone() for k, v in obs["sensor_data"]["base_camera"].items()}
    state0 = env.state_obs.clone()
    snap = env.scene.get_state()
    env.capture_graph()
    env.enable_host_io()
    torch.cuda.synchronize()
    for k in env.scene.STATE_FIELDS:
        assert torch.equal(getattr(env.scene, k), snap[k]), k
    assert torch.equal(env.state_obs, state0)
    for k, v in obs["sensor_data"]["base_camera"].items():
        assert torch.equal(v, st0[k]), k


def test_final_obs_is_the_pre_reset_observation(cuda):
    """info["final_obs"]: for envs auto-reset this step, the state obs of the state the episode
    ended in (what a learner bootstraps from on truncation) == the obs of the same run without
    auto-reset."""
    from paper_2410_00425_b200.metrics import eval_wrapper
    from paper_2410_00425_b200.tasks import make_task

    a = make_task("PickCube", 64, seed=5, overrides={"max_steps": 3})
    b = eval_wrapper(make_task("PickCube", 64, seed=5, overrides={"max_steps": 3}))
    for t in range(3):
        ra = a.step_random(t)
        rb = b.step_random(t)
    # envs that reached the time limit (no early termination on the way) followed the same
    # trajectory in both runs
    done = ra.truncated.bool() & ~ra.terminated.bool()
    assert int(done.sum()) >= 32
    assert torch.equal(ra.info["final_obs"][done], rb.obs[done])
    assert not torch.equal(ra.obs, rb.obs)  # a's obs are the reset states
