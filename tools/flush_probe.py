"""Cold vs warm L2 for the C2 step kernel: bench.measure() with the 256 MiB L2 flush before every
timed step, and with a 4-byte 'flush' (L2 stays warm: state, model tables and the kernel's code).
Also flushing only data: a flush, then one untimed tiny launch of the same kernel family is not
possible without side effects, so the split between code and data misses comes from the ncu
no_instruction stalls.  python tools/flush_probe.py [envs]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_00425_b200.tasks import make_task  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = make_task("PickCube", N, seed=0)
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tiny = torch.empty(4, dtype=torch.uint8, device="cuda")
for rep in range(2):
    for name, fl in (("L2 flushed", big), ("L2 warm", tiny)):
        m = bench.measure(env, 200, 5, fl, None, 0, seed_step=1000 * rep)
        print(f"{name:12s} k_step {m['sim_ms'] / 200 * 1e3:6.1f} us")

# code vs data: after the flush, one 8-env step of a second PickCube env through the SAME kernel
# variant (BS_STEP_G=8 forces it) re-warms the kernel's code in L2 but not this env's state
import os  # noqa: E402
if os.environ.get("BS_STEP_G") == "8":
    import time  # noqa: E402
    small = make_task("PickCube", 8, seed=1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
    for mode in ("flush", "flush + code warm-up"):
        for k in range(200):
            env.random_actions(5000 + k)
            small.random_actions(5000 + k)
            big.zero_()
            if mode != "flush":
                small.launch_step()
            ev[k][0].record()
            env.launch_step()
            ev[k][1].record()
        torch.cuda.synchronize()
        print(f"{mode:22s} k_step {sum(a.elapsed_time(b) for a, b in ev) / 200 * 1e3:6.1f} us")
