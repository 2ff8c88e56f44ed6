"""Splits Env.step_host's per-step cost on a GPU box: full call, without the host-side finite
check, graph replay + sync only, and the device step alone.  python tools/e2e_probe.py [envs]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_00425_b200.tasks import make_task  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = make_task("PickCube", N, seed=0)
env.enable_host_io()
acts = np.random.default_rng(0).uniform(-1, 1, (64, N, 3)).astype(np.float32)
cold = np.random.default_rng(1).uniform(-1, 1, (400, N, 3)).astype(np.float32)  # bench-like: fresh rows


def timeit(fn, n=400):
    for k in range(20):
        fn(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(n):
        fn(k)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print(f"step_host (validated)      {timeit(lambda k: env.step_host(acts[k % 64])):7.1f} us")
print(f"step_host (cold actions)   {timeit(lambda k: env.step_host(cold[k % 400])):7.1f} us")
env.validate_actions = False
print(f"step_host (no finite check){timeit(lambda k: env.step_host(acts[k % 64])):7.1f} us")
stream = torch.cuda.current_stream()
print(f"graph replay + sync        {timeit(lambda k: (env._host_graph.replay(), stream.synchronize())):7.1f} us")
print(f"graph replay only (async)  {timeit(lambda k: env._host_graph.replay()):7.1f} us")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for k in range(100):
    env._host_graph.replay()
ev1.record()
torch.cuda.synchronize()
print(f"graph device time          {ev0.elapsed_time(ev1) * 10:7.1f} us")
a = acts[0]
print(f"python: shape+params key   {timeit(lambda k: (a.shape == (N, 3), env._params_key())):7.2f} us")
print(f"python: raw stream         {timeit(lambda k: torch._C._cuda_getCurrentRawStream(0)):7.2f} us")
print(f"python: current_stream    {timeit(lambda k: torch.cuda.current_stream(env.device).cuda_stream):7.2f} us")
print(f"python: a.ctypes.data      {timeit(lambda k: a.ctypes.data):7.2f} us")
