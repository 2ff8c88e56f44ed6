"""Benchmark: env-steps/s of the PickCube-style tabletop task (BASELINE.json configs[1], "C2":
state obs, 4096 envs per GPU, sim 120 Hz / control 60 Hz, 4 position iterations) on N B200s,
next to the reference CPU path timed on the host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N>1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...)

One "step" = one env.step over every env on every GPU (controller -> 2 substeps of dynamics,
contacts, PGS -> FK -> reward/termination -> state obs -> auto-reset), fed by 1000-style
uniform random actions.  Timing rules:
  * `value`: device time (CUDA events on the launching stream) summed over K steps, inputs
    resident in HBM; the L2 is flushed (256 MiB write) BEFORE every timed step, outside
    the events, so every step starts cold.  Max over ranks; whole-job env-steps/s.
  * `e2e`: the public API (`Env.step(host action)`) with the action copied from pinned
    host memory and obs + reward copied back every step; wall clock, synchronised.
  * `roofline`: the fused step kernel alone (events around its launch), algorithmic bytes
    per env-step / duration vs MEASURED_PEAKS.json hbm_gbs.
  * `cpu_baseline` (rank 0, N=1 only): the oracle (CPU restatement of the reference path,
    numpy) on all host cores, one process per core, for ~10 s.
The reference arm (`--impl reference`) times that same CPU path per step on the same
workload.  NCCL is used only after the timed region, for rollout statistics.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ENVS_PER_GPU = 4096
METRIC = "env-steps/s (sim+render, whole box)"
WORKLOAD = "C2 PickCube-style (ARM3 + cube + ground), obs_mode=state, 4096 envs/GPU"
FALLBACK_HBM_GBS = 6650.0


# ------------------------------------------------------------------------------ helpers
def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        for k in ("hbm_gbs", "hbm_GBs", "hbm"):
            if k in pk:
                return float(pk[k]), "measured"
    except (OSError, ValueError):
        pass
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        time.sleep(0.25)
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(r[0] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": rows[0][1], "reasons": reasons, "samples": len(rows)}


def algorithmic_bytes_per_env_step(scene, obs_dim, action_dim):
    """Bytes the fused step must move per env-step: action read,
    articulation + actor state read and written, drive-target write, goal read/write, obs
    and reward write, flags and counters.  Scratch (link poses, contact rows) is on-chip and
    the link-pose cache write counts as output."""
    D, A, L = scene.models[0].D, scene.models[0].A, scene.models[0].L
    f8 = 8
    b = 4 * action_dim                       # action (f32)
    b += 2 * 2 * D * f8                      # qpos, qvel read + write
    b += D * f8                              # drive targets write
    b += 2 * A * 13 * f8                     # actor pose (7) + vel (6) read + write
    b += 2 * 3 * f8                          # goal read + write
    b += L * 7 * f8                          # link-pose cache write
    b += 4 * obs_dim + 4                     # state obs + reward (f32)
    b += 4 + 4                               # terminated/truncated/success/fail (u8) + unsupported (i32)
    b += 2 * (4 + 4 + 1) + 4 + 4             # elapsed, reset_count, diverged r/w; model_id, target_dof
    return b


# ------------------------------------------------------------------------------ CPU path
def _cpu_worker(args):
    """One host process: the oracle (numpy restatement of the reference path) on a slice of
    envs.  Runs `warmup` steps, waits on the barrier, then `steps` steps (or `seconds`)."""
    (rank, n_envs, env_offset, seed, warmup, steps, seconds, barrier, q) = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    import numpy as np

    from oracle.philox import action_uniforms
    from oracle.tasks import PickCubeOracle
    from paper_2410_00425_b200.descriptors import pickcube_desc, PickCubeSpec

    spec = PickCubeSpec()
    orc = PickCubeOracle(spec, pickcube_desc(spec), n_envs, seed, env_offset=env_offset)
    ids = np.arange(env_offset, env_offset + n_envs)
    for k in range(warmup):
        orc.step(action_uniforms(seed, k, ids, 3))
    barrier.wait()
    t0 = time.perf_counter()
    k = 0
    while True:
        orc.step(action_uniforms(seed, warmup + k, ids, 3))
        k += 1
        if steps is not None and k >= steps:
            break
        if steps is None and time.perf_counter() - t0 >= seconds:
            break
    q.put((rank, k, n_envs, time.perf_counter() - t0))


def cpu_reference(total_envs, warmup, steps=None, seconds=None, seed=0):
    """Time the CPU path with one process per host core.  Returns (env-steps/s, cores, info)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, total_envs))
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(procs)
    q = ctx.Queue()
    per = [total_envs // procs + (1 if r < total_envs % procs else 0) for r in range(procs)]
    offs = [sum(per[:r]) for r in range(procs)]
    ps = [ctx.Process(target=_cpu_worker, args=((r, per[r], offs[r], seed, warmup, steps, seconds, barrier, q),))
          for r in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    if steps is not None:
        t = max(r[3] for r in res)
        rate = total_envs * steps / t
        info = f"{procs} procs x ~{per[0]} envs, {steps} steps of all {total_envs} envs, {t:.1f} s"
    else:
        rate = sum(r[1] * r[2] / r[3] for r in res)
        info = (f"{procs} procs x ~{per[0]} envs ({total_envs} envs total), "
                f"{min(r[1] for r in res)}-{max(r[1] for r in res)} steps each, ~{seconds:.0f} s")
    return rate, procs, info


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    total = ENVS_PER_GPU * args.gpus
    rate, cores, info = cpu_reference(total, args.warmup, steps=args.steps, seed=args.seed)
    ms = total / rate * 1e3
    line = {"metric": METRIC, "value": rate, "unit": "env-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox-seeded resets and actions)",
            "impl": "reference",
            "config": {"workload": WORKLOAD.replace("4096 envs/GPU", f"{total} envs"), "num_envs": total,
                       "sim_freq": 120, "control_freq": 60, "solver_pos_iters": 4, "solver_vel_iters": 0},
            "cpu_baseline": {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "port",
                             "sample": info},
            "e2e": {"value": rate, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU path
def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torch.distributed.run (one rank per GPU)")
    # CPU baseline first (before CUDA is initialised in this process; spawn-based workers)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, cores, info = cpu_reference(ENVS_PER_GPU, 2, seconds=args.cpu_seconds, seed=args.seed)
        cpu = {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "port", "sample": info}

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2410_00425_b200 import _native as nat
    from paper_2410_00425_b200.tasks import make_task

    nat.ensure_device(local)
    n_global = ENVS_PER_GPU * world
    env = make_task("PickCube", n_global, seed=args.seed, shard=(rank, world) if world > 1 else None)
    N = env.num_envs
    dev = env.device
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # ---------------- device-resident throughput (`value`) + step-kernel time (`roofline`)
    for k in range(args.warmup):
        env.step_random(k)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                      # cold L2 before every timed step (not timed)
            ev[k][0].record(stream)
            env.random_actions(args.warmup + k)
            ev[k][1].record(stream)
            env.launch_step()
            ev[k][2].record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = sum(e[0].elapsed_time(e[2]) for e in ev)
    kern_ms = sum(e[1].elapsed_time(e[2]) for e in ev)
    t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, kern_ms = float(t[0]), float(t[1])
    value = n_global * args.steps / (step_ms / 1e3)

    # rollout statistics: the only collective (NCCL all-reduce of a few scalars)
    stats = torch.stack([env.success.sum().double(), env.terminated.sum().double(),
                         env.truncated.sum().double(), env.reward.double().sum()])
    if dist is not None:
        dist.all_reduce(stats)

    # ---------------- end to end through the public API with host buffers (`e2e`)
    import numpy as np

    e2e_steps = max(args.steps, 20)
    rng = np.random.default_rng(args.seed + rank)
    host_actions = torch.from_numpy(rng.uniform(-1, 1, (e2e_steps, N, env.action_dim)).astype(np.float32))
    host_actions = host_actions.pin_memory()
    obs_host = torch.empty((N, env.obs_dim), dtype=torch.float32).pin_memory()
    rew_host = torch.empty((N,), dtype=torch.float32).pin_memory()
    env.capture_graph()
    for k in range(3):
        r = env.step(host_actions[k])
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        r = env.step(host_actions[k])                 # H2D of the action inside
        obs_host.copy_(r.obs, non_blocking=True)      # D2H of the step's results
        rew_host.copy_(r.reward, non_blocking=True)
        stream.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
    e2e = {"value": n_global * e2e_steps / e2e_s, "unit": "env-steps/s",
           "h2d_bytes_per_step": N * env.action_dim * 4, "d2h_bytes_per_step": N * (env.obs_dim + 1) * 4,
           "steps": e2e_steps, "path": "Env.step(pinned host action) + obs/reward D2H, CUDA graph"}

    peak, peak_kind = _peaks()
    bpe = algorithmic_bytes_per_env_step(env.scene, env.obs_dim, env.action_dim)
    kern_s = kern_ms / 1e3 / args.steps
    achieved = bpe * N / kern_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "kernel": "k_step (fused step)", "bytes_per_env_step": bpe,
            "kernel_us_per_launch": kern_s * 1e6, "peak_source": peak_kind}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (Philox-seeded resets and device-generated uniform actions)",
                "config": {"workload": WORKLOAD, "num_envs_per_gpu": ENVS_PER_GPU, "global_envs": n_global,
                           "sim_freq": 120, "control_freq": 60, "solver_pos_iters": 4, "solver_vel_iters": 0,
                           "parallelism": f"env-shard x{world}", "l2": "flushed (256 MiB write) before each timed step"},
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
                "gpu_launches": 2 * args.steps,
                "rollout_stats": {"success": float(stats[0]), "terminated": float(stats[1]),
                                  "truncated": float(stats[2])}}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
