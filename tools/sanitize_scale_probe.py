"""Benchmark-scale workload for compute-sanitizer (tools/sanitize.sh): the persistent rasterizer
with several frames per CTA (frame queue, key-tile reuse across frames) and a full-wave step.

  python tools/sanitize_scale_probe.py [render_envs] [step_envs]
"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2410_00425_b200.tasks import make_task  # noqa: E402

render_envs = int(sys.argv[1]) if len(sys.argv) > 1 else 400   # > 2 x 148 frames: >= 3 per CTA
step_envs = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
env = make_task("PickCube", render_envs, seed=1, obs_mode="rgbd")
env.step_random(0)
env = make_task("OpenCabinet", render_envs // 2, seed=1, obs_mode="pointcloud")
env.step_random(0)
env = make_task("PickCube", step_envs, seed=1)
env.step_random(0)
torch.cuda.synchronize()
print("ok")
