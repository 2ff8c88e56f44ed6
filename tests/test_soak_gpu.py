"""Long-horizon soak of the benchmark workloads on the GPU product: thousands of control steps
with random actions, every episode boundary auto-reset in the kernel.  Nothing may diverge
(a divergent env is flagged and frozen -- it must not happen on these
well-conditioned scenes), every state stays finite and physically bounded, and the episode
bookkeeping is exact (each env completes floor(steps / T) time-limit episodes or more)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("task,n,steps", [("PickCube", 4096, 1500), ("OpenCabinet", 512, 600),
                                          ("PickHetero", 512, 600)])
def test_soak(cuda, task, n, steps):
    from paper_2410_00425_b200.tasks import make_task

    env = make_task(task, n, seed=11)
    env.capture_graph()
    T = env.spec.max_steps
    episodes = torch.zeros(n, dtype=torch.int64, device=env.device)
    for t in range(steps):
        r = env.step_random(t)
        episodes += r.info["episode"]["done"].to(torch.int64)
    torch.cuda.synchronize()
    s = env.scene
    assert int(s.diverged.sum()) == 0
    for k in ("qpos", "qvel", "actor_pose", "actor_vel", "link_pose"):
        assert bool(torch.isfinite(getattr(s, k)).all()), k
    assert float(s.qvel.abs().max()) < 1e3
    if s.A_max:
        ap = s.actor_pose.cpu().numpy()
        assert ap[:, :, 2].min() > -0.05 and np.abs(ap[:, :, :2]).max() < 5.0  # nothing tunnels or flies off
    assert int(episodes.min()) >= steps // T
    assert int(s.elapsed.max()) < T
