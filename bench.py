"""Benchmark: env-steps/s of the PickCube-style tabletop task on N B200s, next to the reference
CPU path timed on the host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c3|c3_4096|c4|c5] [--secondary c3,c3_4096]
  (N>1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...)

Workloads (BASELINE.json configs):
- c2 (the headline, configs[1]): state obs, 4096 envs per GPU;
- c3 (configs[2]): obs_mode rgb+depth (the rasterizer also writes seg on the device), one
  128x128 camera, 1024 envs per GPU;
- c3_4096: the same sim+render workload at the north star's 4096 envs per GPU;
- c4 (configs[3]): OpenCabinet, pointcloud obs from one 128x128 camera, 1024 envs per GPU;
- c5 (configs[4]): PickHetero, rgb+depth+seg from 2 jittered 256x256 cameras, 1024 envs per GPU.
The default run prints the c2 line and attaches c3, c3_4096, c4 and c5 under "secondaries" (every
BASELINE config in one line).

One "step" = one env.step over every env on every GPU. That is: controller -> 2 substeps of
dynamics, contacts and PGS -> FK -> reward/termination -> state obs -> auto-reset, plus the
render for camera workloads. Steps are fed by uniform random actions.

Timing rules:
- `value`: device time (CUDA events on the launching stream, first to last of each step) summed over K steps, with inputs
  resident in HBM. The L2 is flushed (a 256 MiB write) BEFORE every timed step, outside the
  events, so every step starts cold. The max is taken over ranks; the figure is whole-job
  env-steps/s.
- `e2e`: the public API with host buffers (`Env.step_host(host action)`): actions read from
  pinned host memory and obs/reward/flags (+ frames) written back every step; wall clock,
  synchronised, max over ranks.
- `roofline`: the dominant kernel alone (the event pair around its launches inside the timed
  steps). Algorithmic bytes per
  env-step / duration, against
  MEASURED_PEAKS.json hbm_gbs.
- `cpu_baseline` (rank 0, N=1 only): the oracle (CPU restatement of the reference path,
  numpy) on all host cores, one process per core, for a bounded sample (stated, with the CPU
  model).
The reference arm (`--impl reference`) times that same CPU path per step on the same
workload (rank 0 only; every config). NCCL is used only after the timed region: the
max-over-ranks timing and the rollout statistics.
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

def _baseline_metric() -> str:
    """The metric string exactly as BASELINE.json names it."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except (OSError, KeyError, ValueError):
        return "env-steps/s (sim+render, whole box) at 1/2/4/8 B200 vs reference CPU host cores"


METRIC = _baseline_metric()
FALLBACK_HBM_GBS = 6650.0
WORKLOADS = {
    "c2": {"task": "PickCube", "envs": 4096, "obs_mode": "state",
           "desc": "C2 PickCube-style (ARM3 + cube + ground), obs_mode=state, 4096 envs/GPU"},
    "c3": {"task": "PickCube", "envs": 1024, "obs_mode": "rgbd",
           "desc": "C3 PickCube-style, obs_mode=rgb+depth (seg also rendered on the device) 1 camera 128x128, "
                   "1024 envs/GPU"},
    "c3_4096": {"task": "PickCube", "envs": 4096, "obs_mode": "rgbd",
                "desc": "C3 at the north-star scale: PickCube-style sim+render, rgb+depth (seg also rendered) 1 camera "
                        "128x128, 4096 envs/GPU"},
    "c4": {"task": "OpenCabinet", "envs": 1024, "obs_mode": "pointcloud",
           "desc": "C4 OpenCabinet (ARM3 + per-env 2-6 drawer/door cabinet), obs_mode=pointcloud 1 camera "
                   "128x128, 1024 envs/GPU"},
    "c5": {"task": "PickHetero", "envs": 1024, "obs_mode": "rgb+depth+seg",
           "desc": "C5 PickHetero (per-env object kind/size/colour, jittered cameras), rgb+depth+seg 2 cameras "
                   "256x256, 1024 envs/GPU"},
}


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
        self.out = ""

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


def _traffic(kernel: str, workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` on `workload`, from the
    committed ncu --set full capture summary (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(workload, {}).get(kernel)
    except (OSError, ValueError):
        return None


def _issue(kernel: str, workload: str, units: int, launch_s: float, sm_mhz):
    """The instruction-issue side of the roofline (the kernels are latency / issue bound, not
    HBM bound): warp instructions per launch from the committed ncu counters
    (profiles/issue.json, tools/ncu_issue.py; scaled to this launch's env / frame count) over the
    issue capacity of the launch measured here, 4 SMSPs x SMs x SM clock x launch time; plus the
    fp64 FLOP rate (thread-level DFMA x 2 + DADD + DMUL, replicated lanes included) against the
    fp64 pipe's 64 DFMA / SM / clock.  None without a capture for this workload."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            doc = json.load(f)
        rec = (doc.get(workload) or doc[workload.split("_")[0]])[kernel]  # c3_4096: the c3 counts, scaled
    except (OSError, ValueError, KeyError):
        return None
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    hz = (sm_mhz or 1965.0) * 1e6
    scale = units / rec["units"]
    inst = rec["warp_inst"] * scale
    flop = (2 * rec["fp64_dfma_thread_ops"] + rec["fp64_dadd_thread_ops"] + rec["fp64_dmul_thread_ops"]) * scale
    slots = 4 * sms * hz * launch_s
    fp64_peak = 64 * 2 * sms * hz
    return {"warp_inst_per_launch": inst, "issue_slots_per_launch": slots, "frac": inst / slots,
            "fp64_tflops": flop / launch_s / 1e12, "fp64_peak_tflops": fp64_peak / 1e12,
            "fp64_frac": flop / launch_s / fp64_peak,
            "ncu_issue_active": rec["ncu_issue_active"], "ncu_fp64_pipe_active": rec["ncu_fp64_pipe_active"],
            "source": "warp-instruction and fp64 thread-op counts per launch from ncu (" + rec["_capture"] +
                      ", scaled by units); launch time measured here; SM clock = the sampled median"}


_PCIE = {}


def pcie_peak_gbs(local: int) -> dict:
    """Measured host<->device copy-engine bandwidth of this box (pinned host memory, 256 MiB,
    best of 5, CUDA events; once per process): the roofline of the `e2e` path, whose per-step
    bytes cross PCIe."""
    if local in _PCIE:
        return _PCIE[local]
    import torch
    dev = torch.device("cuda", local)
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    out = {}
    for name, (dst, src) in (("d2h", (h, d)), ("h2d", (d, h))):
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out[name] = best
    del h, d
    _PCIE[local] = out
    return out


def sim_bytes_per_env_step(scene, obs_dim, action_dim):
    """Algorithmic bytes of one env-step on SURVEY.md section 8(d)'s basis:
    the action read; articulation (qpos, qvel) and actor (pose 7 + vel 6) state read + write;
    the goal read; the state obs + reward written; the four flag bytes; elapsed read + write.
    fp64 state (the reference's sim precision).  Intermediates the engine also writes -- the
    link-pose (FK) cache, drive targets, counters -- are NOT algorithmic: reported separately
    by aux_bytes_per_env_step."""
    D = max(m.D for m in scene.models)
    A = max(m.A for m in scene.models)
    f8 = 8
    b = 4 * action_dim                       # action (f32)
    b += 2 * 2 * D * f8                      # qpos, qvel read + write
    b += 2 * A * 13 * f8                     # actor pose (7) + vel (6) read + write
    b += 3 * f8                              # goal read
    b += 4 * obs_dim + 4                     # state obs + reward (f32)
    b += 4                                   # terminated / truncated / success / fail (u8)
    b += 2 * 4                               # elapsed read + write
    return b


def aux_bytes_per_env_step(scene):
    """Non-algorithmic bytes the fused step also moves: the link-pose cache write, drive
    targets, goal write-back, reset/divergence counters, unsupported-pair count, model/target ids."""
    D = max(m.D for m in scene.models)
    L = max(m.L for m in scene.models)
    return L * 7 * 8 + D * 8 + 3 * 8 + 2 * (4 + 1) + 4 + 4 + 4


def render_bytes_per_env_step(renderer, scene):
    """Frame bytes written per env-step: rgb 3 + depth 4 + seg 2 per pixel (+ pointcloud 24),
    plus the state read the rasterizer needs (link-pose cache, actor poses, camera pose)."""
    b = 0
    for g in renderer.groups:
        px = g["w"] * g["h"] * len(g["cams"])
        b += px * (3 + 4 + 2) + (px * 24 if g["pc"] is not None else 0)
        b += len(g["cams"]) * (7 * 8 + 4 * 4)
    m = scene.models[0]
    b += (m.L + m.A) * 7 * 8
    return b


# ------------------------------------------------------------------------------ CPU path
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _cpu_task(name, n_envs, env_offset, total_envs, seed):
    """The CPU restatement of workload `name` (oracle/: numpy, fp64 dynamics, fp32 raster) for
    the global envs [env_offset, env_offset + n_envs) of a `total_envs` batch.  Returns
    step(k): one env.step of those envs with the k-th Philox action draw, plus their frames."""
    import numpy as np

    from oracle import raster
    from oracle.contacts import shape_world_poses
    from oracle.dynamics import forward_kinematics
    from oracle.model import BODY_ACTOR, Model
    from oracle.philox import action_uniforms
    from paper_2410_00425_b200 import descriptors as Dd
    from paper_2410_00425_b200 import meshes
    from paper_2410_00425_b200.cameras import (CameraConfig, CameraJitter, RenderParams, default_cameras,
                                               look_at, pinhole, randomize_cameras)
    from paper_2410_00425_b200.scene import PackedModel

    wl = WORKLOADS[name]
    ids = np.arange(env_offset, env_offset + n_envs)
    rp = RenderParams()
    light = np.asarray(rp.light_dir, np.float64) / np.linalg.norm(rp.light_dir)
    pc = wl["obs_mode"] == "pointcloud"
    if wl["task"] == "PickCube":
        spec = Dd.PickCubeSpec()
        from oracle.tasks import PickCubeOracle

        orc = PickCubeOracle(spec, Dd.pickcube_desc(spec), n_envs, seed, env_offset=env_offset)
        descs = [Dd.pickcube_desc(spec)] * n_envs
        cams, jitter = default_cameras(), CameraJitter()

        def poses():  # (env -> (model, LP, LQ, AP, AQ))
            LP, LQ = orc.link_poses()
            return [(0, LP[e], LQ[e], orc.st.ap[e], orc.st.aq[e]) for e in range(n_envs)]
    elif wl["task"] == "OpenCabinet":
        from oracle.tasks import OpenCabinetOracle

        spec = Dd.OpenCabinetSpec()
        descs = Dd.opencabinet_descs(spec, total_envs, seed)[env_offset:env_offset + n_envs]
        orc = OpenCabinetOracle(spec, descs, seed, env_offset=env_offset)
        cams, jitter = default_cameras(), CameraJitter()

        def poses():
            out = [None] * n_envs
            for g in orc.groups:
                LP, LQ = forward_kinematics(g["model"], g["st"].q)
                for r, e in enumerate(g["idx"]):
                    out[e] = (e, LP[r], LQ[r], np.zeros((0, 3)), np.zeros((0, 4)))
            return out
    else:  # PickHetero
        from oracle.tasks import PickHeteroOracle

        spec = Dd.PickHeteroSpec()
        descs = Dd.hetero_descs(spec, total_envs, seed)[env_offset:env_offset + n_envs]
        orc = PickHeteroOracle(spec, descs, seed, env_offset=env_offset)
        res = spec.camera_res
        cams = [CameraConfig(n, pose_p=eye, pose_q=look_at(eye, (-0.15, 0.0, 0.02)), **pinhole(res, res, 60.0))
                for n, eye in (("base_camera", (0.15, 0.5, 0.4)), ("side_camera", (0.15, -0.5, 0.4)))]
        jitter = CameraJitter(spec.camera_pos_jitter, spec.camera_rot_jitter, 0.0)

        def poses():
            out = [None] * n_envs
            for idx, o in orc.groups:
                LP, LQ = o.link_poses()
                for r, e in enumerate(idx):
                    out[e] = (e, LP[r], LQ[r], o.st.ap[r], o.st.aq[r])
            return out
    render = None
    if wl["obs_mode"] != "state":
        models = [Model(d) for d in descs] if wl["task"] != "PickCube" else [Model(descs[0])]
        control = spec.control()
        mesh_cache = {}

        def mesh_of(e):
            d = descs[e]
            k = d.key() if hasattr(d, "key") else 0
            if k not in mesh_cache:
                mesh_cache[k] = meshes.model_mesh(PackedModel(d, control).shapes)
            return mesh_cache[k]
        cpose, cintr = randomize_cameras(cams, n_envs, seed, jitter, env_offset)
        colors = [m.s_color[:, :3].astype(np.float32).copy() for m in models]
        if wl["task"] == "PickHetero":
            objs = Dd.hetero_objects(spec, total_envs, seed)[env_offset:env_offset + n_envs]
            for e, (_, _, rgb) in enumerate(objs):
                m = models[e]
                colors[e][[s for s in range(m.S) if m.s_btype[s] == BODY_ACTOR]] = rgb  # the actor's shape

        def render():
            for (mi, LP, LQ, AP, AQ), e in zip(poses(), range(n_envs)):
                m = models[mi]
                SP, SQ = shape_world_poses(m, LP[None], LQ[None], AP[None], AQ[None])
                for c, cam in enumerate(cams):
                    raster.render_frame(mesh_of(e), m.s_seg, SP[0], SQ[0], cpose[e, c, :3], cpose[e, c, 3:],
                                        cintr[e, c], cam.width, cam.height, cam.near, cam.far, colors[mi], light,
                                        rp.ambient, rp.diffuse, rp.background, pc)
    adim = 3

    def step(k):
        orc.step(action_uniforms(seed, k, ids, adim))
        if render is not None:
            render()
    return step


def _cpu_worker(args):
    """One host process: the CPU path on a slice of envs.  Runs `warmup` steps, waits on the
    barrier, then `steps` steps (or `seconds`)."""
    (rank, name, n_envs, env_offset, total_envs, seed, warmup, steps, seconds, barrier, q) = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    one = _cpu_task(name, n_envs, env_offset, total_envs, seed)
    for k in range(warmup):
        one(k)
    barrier.wait()
    t0 = time.perf_counter()
    k = 0
    while True:
        one(warmup + k)
        k += 1
        if steps is not None and k >= steps:
            break
        if steps is None and time.perf_counter() - t0 >= seconds:
            break
    q.put((rank, k, n_envs, time.perf_counter() - t0))


def cpu_reference(name, sample_envs, total_envs, warmup, steps=None, seconds=None, seed=0):
    """Time the CPU path of workload `name` with one process per host core on the global envs
    [0, sample_envs) of a `total_envs` batch.  Returns (env-steps/s, cores, info)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, sample_envs))
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(procs)
    q = ctx.Queue()
    per = [sample_envs // procs + (1 if r < sample_envs % procs else 0) for r in range(procs)]
    offs = [sum(per[:r]) for r in range(procs)]
    ps = [ctx.Process(target=_cpu_worker,
                      args=((r, name, per[r], offs[r], total_envs, seed, warmup, steps, seconds, barrier, q),))
          for r in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    what = (f"all {total_envs} envs" if sample_envs == total_envs else
            f"a sample of {sample_envs} of the workload's {total_envs} envs (global envs 0-{sample_envs - 1})")
    if steps is not None:
        t = max(r[3] for r in res)
        rate = sample_envs * steps / t
        info = f"{procs} procs x ~{per[0]} envs: {steps} steps of {what}, {t:.1f} s"
    else:
        rate = sum(r[1] * r[2] / r[3] for r in res)
        info = (f"{procs} procs x ~{per[0]} envs: {min(r[1] for r in res)}-{max(r[1] for r in res)} steps of "
                f"{what}, ~{seconds:.0f} s")
    return rate, procs, info + f"; CPU: {cpu_model()}"


def cpu_sample_envs(name, total_envs):
    """Bounded CPU sample: every env for state-only workloads; 4 envs per host core for the
    rendering ones (a step over all of them would take tens of seconds)."""
    if WORKLOADS[name]["obs_mode"] == "state":
        return total_envs
    return min(total_envs, 4 * len(os.sched_getaffinity(0)))


def config_for(name, world):
    """The `config` dict of a workload: identical in both arms (the driver compares them)."""
    wl = WORKLOADS[name]
    return {"workload": wl["desc"], "num_envs_per_gpu": wl["envs"], "global_envs": wl["envs"] * world,
            "obs_mode": wl["obs_mode"], "sim_freq": 120, "control_freq": 60, "solver_pos_iters": 4,
            "solver_vel_iters": 0, "parallelism": f"env-shard x{world}",
            "l2": "flushed (256 MiB write) before each timed GPU step; inputs resident"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    total = WORKLOADS[args.config]["envs"] * args.gpus
    sample = cpu_sample_envs(args.config, total)
    rate, cores, info = cpu_reference(args.config, sample, total, args.warmup, steps=args.steps, seed=args.seed)
    ms = total / rate * 1e3
    line = {"metric": METRIC, "value": rate, "unit": "env-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox-seeded resets and actions)",
            "impl": "reference", "config": config_for(args.config, args.gpus),
            "cpu_baseline": {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "port",
                             "sample": info},
            "e2e": {"value": rate, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU path
def measure(env, steps, warmup, flush, dist, local, seed_step=0):
    """Device timing of `steps` env steps: the steps' synthetic actions are generated into HBM
    before the timed region (Philox, the same stream step_random uses); per step, flush L2
    (untimed), then CUDA events on the launching stream: one before the fused step kernel, one
    after it, and -- render workloads only -- one after the render launches.  The step interval
    is first event -> last event; the kernel intervals are the consecutive pairs.  (An extra
    event record before a kernel costs ~2.5 us of device time per step, so there is none.)"""
    import torch

    from paper_2410_00425_b200 import dist as bdist

    stream = torch.cuda.current_stream(env.device)
    for k in range(warmup):
        env.step_random(seed_step + k)
    acts = torch.empty((steps,) + tuple(env.action_buf.shape), dtype=env.action_buf.dtype, device=env.device)
    for k in range(steps):
        env.random_actions(seed_step + warmup + k)
        acts[k].copy_(env.action_buf)
    torch.cuda.synchronize()
    render = env.renderer is not None
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3 if render else 2)] for _ in range(steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(steps):
            flush.zero_()                      # cold L2 before every timed step (not timed)
            ev[k][0].record(stream)
            env._launch_sim(acts[k].data_ptr())
            ev[k][1].record(stream)
            if render:
                env._render()
                ev[k][2].record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([sum(e[0].elapsed_time(e[-1]) for e in ev), sum(e[0].elapsed_time(e[1]) for e in ev),
                      sum(e[1].elapsed_time(e[2]) for e in ev) if render else 0.0], dtype=torch.float64,
                     device=env.device)
    bdist.max_over_ranks(t)  # the job is as slow as its slowest rank
    # k_step, and per camera group k_frame_setup + k_render (our kernels in the timed region)
    launches = 1 + (2 * len(env.renderer.groups) if render else 0)
    return {"step_ms": float(t[0]), "sim_ms": float(t[1]), "render_ms": float(t[2]), "clocks": clk.summary(),
            "launches": launches * steps}


def measure_e2e(env, steps, dist, seed):
    """The public API with host buffers: Env.step_host(host action) -- one CUDA graph in which
    the step kernel reads the pinned host actions and writes obs / reward / flags to pinned host
    memory over PCIe (zero-copy), plus the render and the D2H copies of the frames -- then a
    stream synchronisation, every step."""
    import numpy as np
    import torch

    from paper_2410_00425_b200 import dist as bdist

    N = env.num_envs
    rng = np.random.default_rng(seed)
    host_actions = rng.uniform(-1, 1, (steps, N, env.action_dim)).astype(np.float32)
    env.enable_host_io()
    for k in range(3):
        env.step_host(host_actions[k])
    h2d, d2h = env.host_io_bytes()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(steps):
        out = env.step_host(host_actions[k])
        _ = out["reward"]
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        e2e_s = float(bdist.max_over_ranks(torch.tensor([e2e_s], dtype=torch.float64, device=env.device))[0])
    return e2e_s, h2d, d2h


def _flatten(d, prefix=""):
    out = {}
    for k, v in d.items():
        if isinstance(v, dict):
            out.update(_flatten(v, prefix + k + "/"))
        else:
            out[prefix + k] = v
    return out


def run_workload(name, steps, warmup, world, rank, local, dist, flush, seed, e2e_steps, cpu):
    import torch

    from paper_2410_00425_b200 import dist as bdist
    from paper_2410_00425_b200.tasks import make_task

    wl = WORKLOADS[name]
    n_global = wl["envs"] * world
    env = make_task(wl["task"], n_global, seed=seed, obs_mode=wl["obs_mode"],
                    shard=(rank, world) if world > 1 else None)
    N = env.num_envs
    m = measure(env, steps, warmup, flush, dist, local)
    value = n_global * steps / (m["step_ms"] / 1e3)
    stats = torch.stack([env.success.sum().double(), env.terminated.sum().double(), env.truncated.sum().double()])
    bdist.reduce_stats(stats)  # rollout statistics: the only data collective
    e2e_s, h2d, d2h = measure_e2e(env, e2e_steps, dist, seed + rank)
    pcie = pcie_peak_gbs(local)
    # the e2e path's own roofline: its per-step host<->device bytes over the measured copy-engine
    # bandwidth (the bytes of one step cross PCIe in sequence: actions in, results out)
    io_gbs = (h2d + d2h) * (e2e_steps / e2e_s) / 1e9
    io_peak = 1.0 / (h2d / (pcie["h2d"] * 1e9) + d2h / (pcie["d2h"] * 1e9)) * (h2d + d2h) / 1e9 if h2d + d2h else None
    e2e_roof = {"bound": "pcie", "achieved": io_gbs, "peak": io_peak, "unit": "GB/s",
                "frac": io_gbs / io_peak if io_peak else None, "pcie_measured_gbs": pcie,
                "source": "h2d/d2h bytes per step x steps/s over the measured pinned copy bandwidth"}
    e2e = {"value": n_global * e2e_steps / e2e_s, "unit": "env-steps/s", "roofline": e2e_roof,
           "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": e2e_steps,
           "path": "Env.step_host: one CUDA graph per step = step kernel reading the pinned host actions and "
                   "writing obs/reward/flags to pinned host memory over PCIe (zero-copy) (+ render + D2H of "
                   "the frames); stream sync every step"}
    peak, peak_kind = _peaks()
    sim_b = sim_bytes_per_env_step(env.scene, env.obs_dim, env.action_dim)
    sim_s = m["sim_ms"] / 1e3 / steps
    kernels = {"k_step": {"us_per_launch": sim_s * 1e6, "bytes_per_env_step": sim_b,
                          "achieved_gbs": sim_b * N / sim_s / 1e9,
                          "aux_bytes_per_env_step": aux_bytes_per_env_step(env.scene)}}
    dominant = "k_step"
    if env.renderer is not None:
        rb = render_bytes_per_env_step(env.renderer, env.scene)
        rs = m["render_ms"] / 1e3 / steps
        kernels["k_render"] = {"us_per_launch": rs * 1e6, "bytes_per_env_step": rb, "achieved_gbs": rb * N / rs / 1e9}
        if rs > sim_s:
            dominant = "k_render"
    dk = kernels[dominant]
    sm_mhz = m["clocks"].get("sm_mhz")
    for k, v in kernels.items():
        v["issue"] = _issue(k, name, N, v["us_per_launch"] / 1e6, sm_mhz)
    roof = {"bound": "hbm", "achieved": dk["achieved_gbs"], "peak": peak, "unit": "GB/s",
            "frac": dk["achieved_gbs"] / peak, "traffic": _traffic(dominant, name), "kernel": dominant,
            "bytes_per_env_step": dk["bytes_per_env_step"], "kernel_us_per_launch": dk["us_per_launch"],
            "peak_source": peak_kind, "issue": dk["issue"], "kernels": kernels}
    line = {"metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": m["step_ms"] / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Philox-seeded resets; device-generated uniform actions, resident in HBM before the timed region)",
            "config": config_for(name, world),
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": m["clocks"],
            "gpu_launches": m["launches"],
            "rollout_stats": {"success": float(stats[0]), "terminated": float(stats[1]), "truncated": float(stats[2])}}
    del env
    torch.cuda.empty_cache()
    return line


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N>1 must be launched with torch.distributed.run (one rank per GPU)")
    # CPU baselines first (before CUDA is initialised in this process; spawn-based workers):
    # rank 0 at N=1 only, a bounded sample of each workload (cpu_sample_envs)
    secondaries = [w for w in (args.secondary or "").split(",") if w and w != args.config]
    cpus = {}
    if rank == 0 and world == 1 and not args.no_cpu:
        for k, name in enumerate([args.config] + secondaries):
            total = WORKLOADS[name]["envs"]
            rate, cores, info = cpu_reference(name, cpu_sample_envs(name, total), total, 1 if k else 2,
                                              seconds=args.cpu_seconds if k == 0 else args.cpu_seconds / 2,
                                              seed=args.seed)
            cpus[name] = {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "port", "sample": info}

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: multi-rank smoke on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2410_00425_b200 import _native as nat
    from paper_2410_00425_b200 import dist as bdist

    nat.ensure_device(local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=torch.device("cuda", local))
    line = run_workload(args.config, args.steps, args.warmup, world, rank, local, dist, flush, args.seed,
                        max(args.steps, 20), cpus.get(args.config))
    line["communicator"] = bdist.describe()
    secs = []
    for name in secondaries:
        sec = run_workload(name, max(args.steps // 4, 20), max(args.warmup, 3), world, rank, local, dist,
                           flush, args.seed, 20, cpus.get(name))
        secs.append({k: sec[k] for k in ("value", "unit", "ms_per_step", "steps", "config", "e2e", "roofline",
                                         "cpu_baseline", "clocks", "gpu_launches")})
    if secs:
        line["secondary"] = secs[0]          # the first extra workload (kept for older readers)
        line["secondaries"] = secs
    if rank == 0:
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
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--secondary", default="c3,c3_4096,c4,c5",
                    help="comma list of extra workloads measured after the headline ('' = none)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--envs", type=int, default=0, help="override envs per GPU (experiments only)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.envs:
        WORKLOADS[args.config] = dict(WORKLOADS[args.config], envs=args.envs,
                                      desc=WORKLOADS[args.config]["desc"] + f" [override: {args.envs} envs/GPU]")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
