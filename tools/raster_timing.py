"""Developer tool: per-phase clocks of the rasterizer (k_render) on the C3 workload.

Run on a GPU box; rebuilds the library with -DBS_PHASE_TIMING (thread 0 of CTAs (0, 0),
(0, 511), (0, 1023) print clock64() deltas at each phase barrier), renders a few C3 frames
batches and prints the mean cycles per phase.  Rebuild normally afterwards.

    python tools/raster_timing.py [envs] [config] [ablate: comma list of rgb,depth,seg,pointcloud]
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["transforms", "vertices", "triangles+live", "tile clear", "classify", "rows+tiny+pixels",
         "resolve after 1st iteration", "resolve 1st iteration (thread 0)"]

CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2410_00425_b200.tasks import make_task
task = {"c3": "PickCube", "c5": "PickHetero", "c4": "OpenCabinet"}[%r]
mode = "pointcloud" if task == "OpenCabinet" else "rgbd"
env = make_task(task, %d, seed=0, obs_mode=mode)
for t in range(3):
    env.step_random(t)
    torch.cuda.synchronize()
if %r:  # output ablation: drop some frame outputs (NULL pointers skip them)
    for g in env.renderer.groups:
        for k in %r.split(","):
            setattr(g["c_out"], k, None)
    print("ABLATE", %r, flush=True)
    for t in range(3):
        env.renderer.render()
        torch.cuda.synchronize()
'''


def main():
    envs = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c3"
    env_vars = dict(os.environ, BS_PHASE_TIMING="1")
    subprocess.run([sys.executable, "-m", "paper_2410_00425_b200.build_native", "--force"], check=True,
                   env=env_vars, cwd=ROOT)
    ablate = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, envs, ablate, ablate, ablate)],
                         capture_output=True, text=True, env=env_vars, cwd=ROOT).stdout
    if ablate:
        out = out.split("ABLATE")[1]
    rows = [list(map(int, l.split()[1:])) for l in out.splitlines() if l.startswith("RTCLK")]
    if not rows:
        print(out)
        raise SystemExit("no RTCLK lines")
    n = len(rows)
    mean = [sum(r[k + 1] for r in rows) / n for k in range(8)]
    tot = sum(mean)
    print(f"{cfg}: {n} samples, {tot:.0f} cycles per frame ({tot / 1.965e3:.1f} us at 1965 MHz)")
    for name, v in zip(NAMES, mean):
        print(f"  {name:20s} {v:9.0f} cycles  {100 * v / tot:5.1f}%")
    if os.environ.get("BS_KEEP_TIMING_BUILD") is None:
        subprocess.run([sys.executable, "-m", "paper_2410_00425_b200.build_native", "--force"], check=True,
                       env={k: v for k, v in os.environ.items() if k != "BS_PHASE_TIMING"}, cwd=ROOT)


if __name__ == "__main__":
    main()
