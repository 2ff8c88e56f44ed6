"""Developer tool: device time of one Renderer.render() (k_frame_setup + k_render) on a fixed
scene -- the env is stepped RT_STEPS times, then the same state is rendered REPS times, each
call timed with CUDA events on the render stream; prints the median and the 10/90 percentiles.

    BS_LIB_PATH=... python tools/render_bench.py [c3|c4|c5] [envs] [steps] [reps]
Used for same-box library A/B runs (tools/gpu_lib_ab.sh times whole bench steps)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_00425_b200.tasks import make_task  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
envs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 200
task, mode = {"c3": ("PickCube", "rgbd"), "c4": ("OpenCabinet", "pointcloud"),
              "c5": ("PickHetero", "rgb+depth+seg")}[cfg]
env = make_task(task, envs, seed=0, obs_mode=mode)
for t in range(steps):
    env.step_random(t)
torch.cuda.synchronize()
r = env.renderer
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for _ in range(5):
    r.render()
torch.cuda.synchronize()
for a, b in ev:
    a.record()
    r.render()
    b.record()
torch.cuda.synchronize()
us = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
lib = os.path.basename(os.environ.get("BS_LIB_PATH", "in-tree"))
print(f"{lib:14s} {cfg} envs={envs} step={steps}: median {np.median(us):8.1f} us  "
      f"p10 {np.percentile(us, 10):8.1f}  p90 {np.percentile(us, 90):8.1f}")
if os.environ.get("RB_SERIES"):
    print("series:", " ".join(f"{v:.0f}" for v in us))
