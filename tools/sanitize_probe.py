"""Small step workload for compute-sanitizer (tools/sanitize.sh): a few control steps of each task."""
import sys, torch
sys.path.insert(0, '.')
from paper_2410_00425_b200.tasks import make_task
for name in (sys.argv[1:] or ["PickCube"]):
    env = make_task(name, 8, seed=1)
    for t in range(3):
        env.step_random(t)
    torch.cuda.synchronize()
print("ok")
