"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path: env sharding, shard
invariance of every per-env random stream, and the statistics collectives (SPEC.md:216, 221,
588).  The step itself is never collective; these are the only
cross-rank operations bench.py performs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.philox import action_uniforms
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200 import dist as bdist
    from paper_2410_00425_b200.cameras import CameraJitter, default_cameras, randomize_cameras
    from paper_2410_00425_b200.descriptors import OpenCabinetSpec, PickCubeSpec, cabinet_kinds, pickcube_desc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    N, seed = 10, 3
    lo, hi = bdist.shard_range(N, rank, WORLD)
    # per-env streams keyed by the global env index
    pose, intr = randomize_cameras(default_cameras(), hi - lo, seed, CameraJitter(0.02, 0.035, 0.05), env_offset=lo)
    kinds = cabinet_kinds(OpenCabinetSpec(), hi - lo, seed, env_offset=lo)
    spec = PickCubeSpec()
    orc = PickCubeOracle(spec, pickcube_desc(spec), hi - lo, seed, env_offset=lo)
    ids = np.arange(lo, hi)
    for t in range(5):
        orc.step(action_uniforms(seed, t, ids, 3))
    snap = orc.snapshot()
    # statistics collectives
    stats = torch.tensor([rank + 1.0, 10.0 * (rank + 1), 5.0, 1.0, 0.0, rank, 0.0], dtype=torch.float64)
    bdist.reduce_stats(stats)
    tmax = bdist.max_over_ranks(torch.tensor([1.0 + rank, 3.0 - rank], dtype=torch.float64))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=lo, hi=hi, pose=pose, intr=intr,
             kinds=np.array(kinds), q=snap["q"], ap=snap["ap"], stats=stats.numpy(), tmax=tmax.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_collectives(tmp_path):
    from oracle.philox import action_uniforms
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.cameras import CameraJitter, default_cameras, randomize_cameras
    from paper_2410_00425_b200.descriptors import OpenCabinetSpec, PickCubeSpec, cabinet_kinds, pickcube_desc

    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    r = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(WORLD)]
    assert (int(r[0]["lo"]), int(r[0]["hi"]), int(r[1]["lo"]), int(r[1]["hi"])) == (0, 5, 5, 10)
    # shards concatenate to the single-process batch, bitwise
    N, seed = 10, 3
    pose, intr = randomize_cameras(default_cameras(), N, seed, CameraJitter(0.02, 0.035, 0.05))
    assert np.array_equal(np.concatenate([x["pose"] for x in r]), pose)
    assert np.array_equal(np.concatenate([x["intr"] for x in r]), intr)
    assert list(np.concatenate([x["kinds"] for x in r])) == cabinet_kinds(OpenCabinetSpec(), N, seed)
    spec = PickCubeSpec()
    orc = PickCubeOracle(spec, pickcube_desc(spec), N, seed)
    for t in range(5):
        orc.step(action_uniforms(seed, t, np.arange(N), 3))
    assert np.array_equal(np.concatenate([x["q"] for x in r]), orc.snapshot()["q"])
    assert np.array_equal(np.concatenate([x["ap"] for x in r]), orc.snapshot()["ap"])
    # SUM of statistics and MAX of timings are identical on every rank
    for x in r:
        assert np.array_equal(x["stats"], [3.0, 30.0, 10.0, 2.0, 0.0, 1.0, 0.0])
        assert np.array_equal(x["tmax"], [2.0, 3.0])


def test_shard_range_properties():
    from paper_2410_00425_b200.dist import shard_range, summarize

    for n in (1, 7, 4096, 4097):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, k, w) for k in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[k][1] == rs[k + 1][0] for k in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    s = summarize(torch.tensor([4.0, -8.0, 400.0, 2.0, 1.0, 1.0, 0.0], dtype=torch.float64))
    assert s["episodes"] == 4 and s["mean_return"] == -2.0 and s["success_once"] == 0.5
