"""The product's N>1 path on one GPU: two ranks (gloo for the collectives, both on cuda:0) each
build their env shard with make_task(..., shard=(rank, 2)), step it with the device Philox
actions, and all-gather the state rows; the concatenation must equal a 1-rank run of the same
global batch BITWISE (no cross-env coupling, RNG keyed by the global env).
The rollout statistics go through dist.reduce_stats and the timing through max_over_ranks --
the collectives bench.py uses under torchrun."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD, N, SEED, STEPS = 2, 64, 3, 30
FIELDS = ("qpos", "qvel", "actor_pose", "actor_vel", "goal", "elapsed", "reset_count", "link_pose")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, port, out_dir, task):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2410_00425_b200 import dist as bdist
    from paper_2410_00425_b200.tasks import make_task

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    env = make_task(task, N, seed=SEED, shard=(rank, WORLD))
    lo, hi = bdist.shard_range(N, rank, WORLD)
    assert env.scene.env_offset == lo and env.num_envs == hi - lo
    done = torch.zeros((), dtype=torch.float64, device=env.device)
    for t in range(STEPS):
        r = env.step_random(t)
        done += (r.terminated | r.truncated).sum().double()
    torch.cuda.synchronize()
    stats = bdist.reduce_stats(torch.stack([done, torch.tensor(float(env.num_envs), device=env.device,
                                                                dtype=torch.float64)]))
    tmax = bdist.max_over_ranks(torch.tensor([float(rank)], dtype=torch.float64, device=env.device))
    parts = {}
    for k in FIELDS:
        local = getattr(env.scene, k).cpu().contiguous()
        gathered = [torch.empty_like(local) for _ in range(WORLD)]
        dist.all_gather(gathered, local)
        parts[k] = torch.cat(gathered).numpy()
    if rank == 0:
        np.savez(os.path.join(out_dir, "gathered.npz"), stats=stats.cpu().numpy(), tmax=tmax.cpu().numpy(),
                 desc=np.array([str(bdist.describe())]), **parts)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("task", ["PickCube", "OpenCabinet"])
def test_two_rank_shards_equal_one_rank_run(cuda, tmp_path, task):
    from paper_2410_00425_b200.tasks import make_task

    mp.spawn(_rank, args=(_free_port(), str(tmp_path), task), nprocs=WORLD, join=True)
    got = dict(np.load(tmp_path / "gathered.npz"))
    full = make_task(task, N, seed=SEED)
    done = 0
    for t in range(STEPS):
        r = full.step_random(t)
        done += int((r.terminated | r.truncated).sum())
    torch.cuda.synchronize()
    for k in FIELDS:
        assert np.array_equal(got[k], getattr(full.scene, k).cpu().numpy()), k
    assert got["stats"][0] == done and got["stats"][1] == N  # SUM over ranks
    assert got["tmax"][0] == WORLD - 1  # MAX over ranks
    assert "gloo" in str(got["desc"][0])
