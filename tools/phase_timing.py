"""Developer tool: split the fused step's per-env critical path into its phases.

Run on a GPU box (it rebuilds the library with -DBS_PHASE_TIMING first):

    python tools/phase_timing.py [envs] [steps] [task]

Thread 0 of CTA 0 records clock64() deltas at each phase boundary of k_step. Every env's step
runs the same phase sequence and the kernel is latency-bound (k_step time is flat from 1024 to
4096 envs, profiles/r01_summary.md). One warp's phase split is therefore the kernel's. The tool
prints cycles per step and the share of each phase, and writes JSON to
gpurun_out/phase_timing.json.
"""

import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {0: "launch/param load", 1: "stage state + controller", 2: "FK (lanes + lane-0 chain)",
         3: "A: subspaces, inertias, shape poses, free bodies", 4: "B: RNEA forward (lane 0)",
         5: "C: link forces", 6: "D: RNEA backward + composite (lane 0)", 7: "E: CRBA",
         8: "F: drives + Cholesky (lane 0)", 9: "G: M^-1 columns", 10: "H: narrowphase",
         11: "I: compaction", 12: "J: constraint rows", 13: "K: PGS sweeps", 14: "L: integrate + limits",
         15: "final FK", 16: "task eval + auto-reset", 17: "write-back + obs"}


def main():
    envs = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    env_vars = dict(os.environ, BS_PHASE_TIMING="1")
    subprocess.run([sys.executable, "-m", "paper_2410_00425_b200.build_native", "--force"], check=True, env=env_vars,
                   cwd=ROOT)
    import torch

    from paper_2410_00425_b200 import _native as nat
    from paper_2410_00425_b200.tasks import make_task

    task = sys.argv[3] if len(sys.argv) > 3 else "PickCube"
    env = make_task(task, envs, seed=0)
    for k in range(5):
        env.step_random(k)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 32)()
    nat.call("bs_debug_phase_clocks", ctypes.addressof(buf), 32, 1)  # reset
    # PHASE_FLUSH=1: a 256 MiB write before every timed step (cold L2, as in bench.py)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("PHASE_FLUSH") else None
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        env.step_random(100 + k)
    torch.cuda.synchronize()
    nat.call("bs_debug_phase_clocks", ctypes.addressof(buf), 32, 0)
    vals = {i: buf[i] / steps for i in range(18)}
    vals[0] = 0.0  # the first tick of a launch measures the gap since the previous launch
    tot = sum(vals.values())
    out = {"task": task, "envs": envs, "steps": steps, "cycles_per_step": tot,
           "phases": {NAMES[i]: {"cycles": v, "share": v / tot} for i, v in vals.items() if i in NAMES}}
    for i, v in sorted(vals.items(), key=lambda x: -x[1]):
        print(f"{v:10.0f} cyc  {100 * v / tot:5.1f}%  {NAMES.get(i, i)}")
    print(f"total {tot:.0f} cycles per step ({tot / 1.965e3:.1f} us at 1965 MHz)")
    subs = 2 * steps  # substeps per step (sim 120 Hz / control 60 Hz)
    out["contacts_env0_per_substep"] = buf[20] / subs
    out["contacts_warp_max_per_substep"] = buf[21] / subs
    print(f"contacts per substep: env0 {buf[20] / subs:.2f}, warp max {buf[21] / subs:.2f}")
    if buf[24]:
        mean_cta = buf[23] / buf[24]
        print(f"per-CTA duration over all launches: mean {mean_cta:.0f} cycles, max {buf[22]:.0f} cycles "
              f"({buf[22] / 1.965e3:.1f} us) -- the launch lasts as long as its slowest warp")
        out["cta_cycles_mean"], out["cta_cycles_max"] = mean_cta, buf[22]
    # launch window: event-timed step kernel vs the CTAs' globaltimer span (entry of the first CTA
    # to exit of the last), one launch at a time
    win = []
    for k in range(20):
        nat.call("bs_debug_phase_clocks", ctypes.addressof(buf), 32, 1)  # reset
        env.random_actions(1000 + k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        env.launch_step()
        e1.record()
        torch.cuda.synchronize()
        nat.call("bs_debug_phase_clocks", ctypes.addressof(buf), 32, 0)
        first = (~buf[25]) & ((1 << 64) - 1)
        win.append((e0.elapsed_time(e1) * 1e3, (buf[26] - first) / 1e3, (buf[27] - first) / 1e3))
    ev = sorted(w[0] for w in win)[len(win) // 2]
    span = sorted(w[1] for w in win)[len(win) // 2]
    ramp = sorted(w[2] for w in win)[len(win) // 2]
    print(f"launch window (median of 20): event-timed step {ev:.1f} us, CTA span (first entry -> last exit) "
          f"{span:.1f} us, CTA entry ramp {ramp:.1f} us")
    out["launch_window_us"] = {"event": ev, "cta_span": span, "entry_ramp": ramp}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "phase_timing.json"), "w") as f:
        json.dump(out, f, indent=1)
    # restore the product build
    subprocess.run([sys.executable, "-m", "paper_2410_00425_b200.build_native", "--force"], check=True,
                   env={k: v for k, v in os.environ.items() if k != "BS_PHASE_TIMING"}, cwd=ROOT)


if __name__ == "__main__":
    main()
