"""Developer tool: per-phase clocks of the rasterizer (k_render) on the C3 workload.

Each phase time is thread 0's clock between consecutive phase barriers (BAR.SYNC may let the
clock read issue before the barrier resolves, so a phase can absorb the previous one's tail).

Run on a GPU box; rebuilds the library with -DBS_PHASE_TIMING (thread 0 of CTAs (0, 0),
(0, 511), (0, 1023) print clock64() deltas at each phase barrier), renders a few C3 frames
batches and prints the mean cycles per phase.  Rebuild normally afterwards.

    [RT_STEPS=n] python tools/raster_timing.py [envs] [config] [ablate: comma list of rgb,depth,seg,pointcloud]
(RT_STEPS: env steps before the measured frames; later steps = the arm farther from rest)
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {1: "transforms", 2: "vertices", 3: "triangles+live", 4: "tile clear", 5: "classify",
         0: "tiny + row spans (4a)", 6: "scan + span walk (4b, 4c)", 7: "resolve"}
ORDER = [1, 2, 3, 4, 5, 0, 6, 7]

CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2410_00425_b200.tasks import make_task
task = {"c3": "PickCube", "c5": "PickHetero", "c4": "OpenCabinet"}[%r]
mode = "pointcloud" if task == "OpenCabinet" else "rgbd"
env = make_task(task, %d, seed=0, obs_mode=mode)
import os
for t in range(int(os.environ.get("RT_STEPS", "3"))):
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
    if os.environ.get("RT_SKIP_FIRST"):  # drop each CTA's first frame (it clears the whole key tile)
        rows = rows[1::3] + rows[2::3] if len(rows) % 3 == 0 else rows
    if not rows:
        print(out)
        raise SystemExit("no RTCLK lines")
    n = len(rows)
    # RTCLK columns: marks 1..7 then 0
    col = {k: k for k in range(1, 8)}
    col[0] = 8
    mean = {k: sum(r[col[k]] for r in rows) / n for k in ORDER}
    tot = sum(mean.values())
    print(f"{cfg}: {n} samples, {tot:.0f} cycles per frame ({tot / 1.965e3:.1f} us at 1965 MHz)")
    for k in ORDER:
        print(f"  {NAMES[k]:28s} {mean[k]:9.0f} cycles  {100 * mean[k] / tot:5.1f}%")
    if os.environ.get("BS_KEEP_TIMING_BUILD") is None:
        subprocess.run([sys.executable, "-m", "paper_2410_00425_b200.build_native", "--force"], check=True,
                       env={k: v for k, v in os.environ.items() if k != "BS_PHASE_TIMING"}, cwd=ROOT)


if __name__ == "__main__":
    main()
