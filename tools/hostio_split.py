"""Where the host-I/O step's device time goes: the step kernel captured four ways -- actions read
from pinned host memory or from HBM, outputs (obs/reward/flags) written to pinned host memory or
to HBM -- each graph replayed back to back (warm L2), device time per step from CUDA events.
python tools/hostio_split.py [envs]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_00425_b200 import _native as nat  # noqa: E402
from paper_2410_00425_b200.tasks import make_task  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = make_task("PickCube", N, seed=0)
env.enable_host_io()
env.step_host(torch.zeros(N, env.action_dim).numpy())
sc = env.scene


def graph(act_ptr, c_out):
    def launch():
        nat.call("bs_step", ctypes.byref(sc.c_tables), ctypes.byref(sc.c_state), ctypes.byref(c_out),
                 ctypes.byref(env.c_params), act_ptr, nat.stream_handle())
    launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        launch()
    return g


variants = {"actions host, outputs host": graph(env._h_action.data_ptr(), env._c_out_host),
            "actions HBM,  outputs host": graph(env.action_buf.data_ptr(), env._c_out_host),
            "actions host, outputs HBM ": graph(env._h_action.data_ptr(), env.c_out),
            "actions HBM,  outputs HBM ": graph(env.action_buf.data_ptr(), env.c_out)}
for rep in range(2):
    for name, g in variants.items():
        for _ in range(10):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / 200 * 1e3:6.1f} us per step (back to back)")
