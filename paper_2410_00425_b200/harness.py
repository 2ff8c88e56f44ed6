"""Throughput benchmark harness (the ``bench`` module; Appendix B).

Reproduces the paper's FPS-vs-env-count methodology on the B200 engine and writes the data
tables behind its scaling figures:

* ``run_bench(task, num_envs_list, steps, camera_setup, warmup_steps)`` -> ``list[BenchResult]``.
  For each env count: build the task, run ``warmup_steps`` random-action steps, then time
  ``steps`` random-action steps.  With cameras, each step also renders every camera and the
  observation tensors are produced ("renders + observation fetches").  Out-of-memory
  becomes a per-setting failure row (fps 0) and the remaining settings continue.
* ``emit_csv(results, path)``: columns exactly ``task,num_envs,steps,wall_seconds,fps,
  peak_rss_bytes,cameras,obs_mode``, rows sorted by (task, cameras, num_envs).
  Floats are written with ``repr`` so parse -> emit round-trips bitwise.
* ``emit_plotdata(results, path)``: JSON series keyed by camera setup.

The timed loop is the engine's own step: one fused ``bs_step`` launch (controller, substeps,
reward, obs, auto-reset) plus, with cameras, one ``bs_render`` launch per resolution.  Random
actions come from the shared Philox stream on the device.  Reward and termination are fused into
the step kernel, so they stay inside the timed region; the paper removes them.
They cost about 2% of ``k_step`` (tools/phase_timing.py), so this makes the numbers slightly
conservative.  ``wall_seconds`` is host wall time around the loop, synchronized on both ends.
``peak_rss_bytes`` is the host's peak resident set (``ru_maxrss``), as the SPEC labels it
(SPEC.md:745); the device's peak allocation is reported beside it in the plot data.

CLI: ``python -m paper_2410_00425_b200.harness run --task PickCube --envs
4,16,64,256,1024 --steps 1000 --cameras 1x640x480 --out results.csv``
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import resource
import sys
import time
from dataclasses import dataclass, field
from typing import Callable, Iterable, List, Optional

CSV_COLUMNS = ("task", "num_envs", "steps", "wall_seconds", "fps", "peak_rss_bytes", "cameras", "obs_mode")
# The paper's ablation grid (Appendix B.3).
CAMERA_SETUPS = ("none", "1x128x128", "1x256x256", "1x512x512", "1x640x480", "3x320x180")


@dataclass
class BenchResult:
    """SPEC.md:716-719.  fps = num_envs * steps / wall_seconds (0 on a failure row)."""

    task: str
    num_envs: int
    steps: int
    wall_seconds: float
    fps: float
    peak_rss_bytes: int
    cameras: str
    obs_mode: str
    error: str = ""                       # failure rows only; not a CSV column
    extra: dict = field(default_factory=dict)  # device peak memory etc. (plot data only)

    def row(self):
        return [self.task, str(self.num_envs), str(self.steps), repr(float(self.wall_seconds)),
                repr(float(self.fps)), str(self.peak_rss_bytes), self.cameras, self.obs_mode]


def fps_of(num_envs: int, steps: int, wall_seconds: float) -> float:
    """fps = num_envs * steps / wall_seconds."""
    if wall_seconds <= 0.0:
        raise ValueError(f"wall_seconds must be positive, got {wall_seconds}")
    return num_envs * steps / wall_seconds


def parse_camera_setup(setup: str):
    """'none' -> []; 'KxWxH' -> K cameras of W x H (width x height, as '1x640x480')."""
    if setup in ("none", "", None):
        return []
    try:
        k, w, h = (int(x) for x in setup.lower().split("x"))
    except ValueError:
        raise ValueError(f"camera setup {setup!r} is not 'none' or 'KxWxH'") from None
    if k < 1 or w < 1 or h < 1:
        raise ValueError(f"camera setup {setup!r} needs positive counts")
    return [(w, h)] * k


def cameras_for(setup: str):
    """CameraConfigs for a setup string: the tabletop view, with K cameras spread on an arc
    around the scene (60 degree vertical field of view)."""
    from .cameras import CameraConfig, look_at, pinhole

    sizes = parse_camera_setup(setup)
    out = []
    target = (-0.15, 0.0, 0.02)
    for i, (w, h) in enumerate(sizes):
        ang = math.radians(90.0 + 50.0 * (i - (len(sizes) - 1) / 2.0))
        eye = (target[0] + 0.6 * math.cos(ang) + 0.3, target[1] + 0.6 * math.sin(ang) - 0.1, 0.4)
        out.append(CameraConfig(f"camera_{i}", pose_p=eye, pose_q=look_at(eye, target), **pinhole(w, h, 60.0)))
    return out


def _peak_rss_bytes() -> int:
    r = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
    return int(r) * (1 if sys.platform == "darwin" else 1024)


def _is_oom(exc: BaseException) -> bool:
    try:
        import torch

        if isinstance(exc, torch.cuda.OutOfMemoryError):
            return True
    except Exception:  # pragma: no cover - torch always importable here
        pass
    return isinstance(exc, MemoryError) or "out of memory" in str(exc).lower()


def run_bench(task: str, num_envs_list: Iterable[int], steps: int = 1000, camera_setup: str = "none",
              warmup_steps: int = 100, obs_mode: Optional[str] = None, seed: int = 0,
              make_env: Optional[Callable] = None, clock: Callable[[], float] = time.perf_counter,
              sync: Optional[Callable[[], None]] = None) -> List[BenchResult]:
    """SPEC.md:720-726.  `make_env(task, num_envs, seed, obs_mode, cameras)` and `clock`/`sync`
    are injectable (tests use a synthetic timer); the defaults build the task on the GPU."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    cams = cameras_for(camera_setup)
    mode = obs_mode or ("rgbd" if cams else "state")
    if mode != "state" and not cams:
        raise ValueError(f"obs_mode {mode!r} needs cameras")
    if make_env is None:
        from .tasks import make_task

        def make_env(t, n, s, m, c):
            return make_task(t, n, seed=s, obs_mode=m, cameras=c or None)

    if sync is None:
        def sync():
            import torch

            torch.cuda.synchronize()

    results = []
    for n in num_envs_list:
        n = int(n)
        env = None
        try:
            env = make_env(task, n, seed, mode, cams)
            for k in range(warmup_steps):
                env.step_random(k)
            sync()
            t0 = clock()
            for k in range(steps):
                env.step_random(warmup_steps + k)
            sync()
            wall = clock() - t0
            extra = {}
            try:
                import torch

                if torch.cuda.is_available():
                    extra["device_peak_bytes"] = int(torch.cuda.max_memory_allocated())
            except Exception:
                pass
            results.append(BenchResult(task, n, steps, wall, fps_of(n, steps, wall), _peak_rss_bytes(),
                                       camera_setup or "none", mode, extra=extra))
        except Exception as exc:  # noqa: BLE001 - OOM rows; anything else propagates
            if not _is_oom(exc):
                raise
            results.append(BenchResult(task, n, steps, 0.0, 0.0, _peak_rss_bytes(), camera_setup or "none", mode,
                                       error=f"out of memory: {str(exc).splitlines()[0][:200]}"))
        finally:
            del env
            try:
                import torch

                if torch.cuda.is_available():
                    torch.cuda.empty_cache()
            except Exception:
                pass
    return results


def _sorted(results):
    return sorted(results, key=lambda r: (r.task, r.cameras, r.num_envs))


def emit_csv(results, path) -> None:
    """exact columns, rows sorted by (task, cameras, num_envs)."""
    results = list(results)
    if not results:
        raise ValueError("emit_csv needs at least one result")
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for r in _sorted(results):
            w.writerow(r.row())


def parse_csv(path) -> List[BenchResult]:
    with open(path, newline="") as f:
        rd = csv.reader(f)
        head = next(rd)
        if tuple(head) != CSV_COLUMNS:
            raise ValueError(f"unexpected columns {head}")
        return [BenchResult(t, int(n), int(s), float(ws), float(fp), int(rss), cam, om)
                for t, n, s, ws, fp, rss, cam, om in rd]


def emit_plotdata(results, path) -> None:
    """JSON series keyed by camera setup."""
    results = list(results)
    if not results:
        raise ValueError("emit_plotdata needs at least one result")
    series = {}
    for r in _sorted(results):
        s = series.setdefault(r.cameras, {"task": [], "num_envs": [], "fps": [], "wall_seconds": [],
                                          "peak_rss_bytes": [], "obs_mode": [], "device_peak_bytes": [],
                                          "error": []})
        s["task"].append(r.task)
        s["num_envs"].append(r.num_envs)
        s["fps"].append(r.fps)
        s["wall_seconds"].append(r.wall_seconds)
        s["peak_rss_bytes"].append(r.peak_rss_bytes)
        s["obs_mode"].append(r.obs_mode)
        s["device_peak_bytes"].append(r.extra.get("device_peak_bytes"))
        s["error"].append(r.error)
    with open(path, "w") as f:
        json.dump(series, f, indent=1, sort_keys=True)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2410_00425_b200.harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="FPS vs number of envs (SPEC.md:741)")
    run.add_argument("--task", default="PickCube")
    run.add_argument("--envs", default="4,16,64,256,1024")
    run.add_argument("--steps", type=int, default=1000)
    run.add_argument("--warmup", type=int, default=100)
    run.add_argument("--cameras", default="none")
    run.add_argument("--obs-mode", default=None)
    run.add_argument("--seed", type=int, default=0)
    run.add_argument("--out", default="results.csv")
    run.add_argument("--plotdata", default=None)
    a = ap.parse_args(argv)
    envs = [int(x) for x in a.envs.split(",") if x]
    res = run_bench(a.task, envs, a.steps, a.cameras, a.warmup, a.obs_mode, a.seed)
    emit_csv(res, a.out)
    if a.plotdata:
        emit_plotdata(res, a.plotdata)
    for r in _sorted(res):
        print(f"{r.task} n={r.num_envs} cams={r.cameras} fps={r.fps:.1f} {r.error}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
