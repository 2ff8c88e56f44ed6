"""Edge cases on the device path: batch sizes that leave idle lane groups, a single env,
partial resets (SPEC.md:536-544 examples), empty pose batches, and argument errors surfaced
as the reference's exception classes."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 5])
def test_odd_batch_sizes_match_oracle(cuda, n):
    from oracle.philox import action_uniforms
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.tasks import make_task, pickcube_scene

    env = make_task("PickCube", n, seed=31)
    orc = PickCubeOracle(env.spec, pickcube_scene(env.spec), n, 31)
    for t in range(8):
        s = env.scene
        ap, av = s.actor_pose.cpu().numpy(), s.actor_vel.cpu().numpy()
        orc.load({"q": s.qpos.cpu().numpy(), "qd": s.qvel.cpu().numpy(), "ap": ap[:, :, :3], "aq": ap[:, :, 3:],
                  "av": av[:, :, :3], "aw": av[:, :, 3:], "goal": s.goal.cpu().numpy(),
                  "elapsed": s.elapsed.cpu().numpy()})
        orc.reset_count[:] = s.reset_count.cpu().numpy().astype(np.uint64)
        env.step_random(t)
        orc.step(action_uniforms(31, t, np.arange(n), 3))
        assert np.abs(env.scene.qpos.cpu().numpy() - orc.snapshot()["q"]).max() < 1e-9


def test_partial_reset_examples(cuda):
    # same seed, full reset twice -> identical obs bitwise; a partial reset of
    # env 0 leaves env 1 bitwise unchanged
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickCube", 4, seed=2)
    o1 = env.reset(seed=2).clone()
    for t in range(5):
        env.step_random(t)
    o2 = env.reset(seed=2).clone()
    assert torch.equal(o1, o2)
    for t in range(5):
        env.step_random(t)
    before = env.scene.get_state()
    obs_before = env.state_obs.clone()
    env.reset(env_mask=torch.tensor([1, 0, 0, 0], dtype=torch.bool))
    after = env.scene.get_state()
    for k in env.scene.STATE_FIELDS:  # every state row, the FK cache included
        assert torch.equal(before[k][1:], after[k][1:]), k
    assert torch.equal(env.state_obs[1:], obs_before[1:])  # re-emitted obs of untouched envs
    assert int(after["elapsed"][0]) == 0 and int(after["reset_count"][0]) == int(before["reset_count"][0]) + 1


def test_empty_pose_batch_and_dimension_errors(cuda):
    from paper_2410_00425_b200 import DimensionError
    from paper_2410_00425_b200.pose import PoseBatch

    a = PoseBatch(np.zeros((0, 3)), np.zeros((0, 4)))
    b = a.compose(a)
    assert b.numpy()[0].shape == (0, 3)
    x = PoseBatch(np.zeros((3, 3)), np.tile([1.0, 0, 0, 0], (3, 1)))
    y = PoseBatch(np.zeros((5, 3)), np.tile([1.0, 0, 0, 0], (5, 1)))
    with pytest.raises(DimensionError, match="3.*5|5.*3"):
        x.compose(y)


def test_bad_action_shapes_and_values(cuda):
    from paper_2410_00425_b200.errors import DimensionError, InputError
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickCube", 2, seed=0)
    with pytest.raises(DimensionError):
        env.step(torch.zeros((3, 3)))
    with pytest.raises(InputError):
        env.step_host(np.full((2, 3), np.inf, np.float32))
    with pytest.raises(DimensionError):
        env.step_host(np.zeros((2, 4), np.float32))
    # one non-finite entry among finite ones is rejected before anything is launched; the
    # largest finite floats are not (the host check is a dot with zeros: no overflow)
    before = env.scene.get_state()
    for bad in (np.nan, -np.inf, np.inf):
        a = np.zeros((2, 3), np.float32)
        a[1, 2] = bad
        with pytest.raises(InputError):
            env.step_host(a)
    after = env.scene.get_state()
    for k in env.scene.STATE_FIELDS:
        assert torch.equal(before[k], after[k]), k
    env.step_host(np.full((2, 3), np.finfo(np.float32).max, np.float32))
    env.step_host(np.full((2, 3), -np.finfo(np.float32).max, np.float32))


def test_time_limit_and_early_termination_examples(cuda):
    """with no early termination, truncated is true exactly at step T; an env in
    its success state with early termination on is terminated that very step."""
    from paper_2410_00425_b200.metrics import eval_wrapper
    from paper_2410_00425_b200.tasks import make_task

    T = 5
    env = eval_wrapper(make_task("PickCube", 4, seed=1, overrides={"max_steps": T}))
    for t in range(1, T + 2):
        r = env.step(torch.zeros((4, 3), device=env.device))
        assert bool(r.truncated.all()) == (t >= T), t
        assert not bool(r.terminated.any())
    env = make_task("PickCube", 4, seed=1)
    s = env.scene
    s.actor_pose[1, 0, :2] = s.goal[1, :2]  # env 1 starts on its goal: success on the next step
    r = env.step(torch.zeros((4, 3), device=env.device))
    assert bool(r.info["success"][1]) and bool(r.terminated[1])
    done = (r.info["success"] | r.info["fail"]).bool()
    assert torch.equal(r.terminated.bool(), done)
