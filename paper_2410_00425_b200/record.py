"""Trajectory recording and deterministic replay.

A TrajectoryFile is a directory: ``manifest.json`` plus one little-endian raw array per field
(SPEC.md:694 container decision).  A recording captures a batched rollout of every env:

- the initial StateSnapshot (``initial/<field>.bin``);
- the action stream ``actions.bin`` (T, N, D) float32;
- per-step success flags ``success.bin`` (T, N) u8;
- optionally the per-step snapshot stream (``states/<field>.bin``, (T, N, ...)).

Everything a replay needs is deterministic on the device, including in-kernel auto-resets
(Philox keyed by global env index and reset count). Replay therefore re-simulates bitwise.
``replay`` can also regenerate observations in another obs mode (e.g. render rgb+depth along
the identical state trajectory) without altering dynamics.
"""

from __future__ import annotations

import dataclasses
import json
import math
import os
import time

import numpy as np
import torch

from . import __version__
from . import _native as nat
from .errors import LayoutMismatchError

STATE_STREAM = ("qpos", "qvel", "actor_pose", "actor_vel", "elapsed", "reset_count", "diverged")


def _write(path, name, arr):
    a = np.ascontiguousarray(arr)
    a.astype(a.dtype.newbyteorder("<")).tofile(os.path.join(path, name + ".bin"))
    return {"shape": list(a.shape), "dtype": a.dtype.str}


def _read(path, name, meta):
    return np.fromfile(os.path.join(path, name + ".bin"), dtype=np.dtype(meta["dtype"])).reshape(meta["shape"])


def record(env, policy, steps: int, path: str, source: str = "policy", store_states: bool = True) -> dict:
    """Roll `policy(obs) -> (N, D) action` for `steps` control steps and write a TrajectoryFile."""
    os.makedirs(os.path.join(path, "initial"), exist_ok=True)
    if store_states:
        os.makedirs(os.path.join(path, "states"), exist_ok=True)
    snap0 = env.scene.get_state()
    obs = env._obs()
    actions, success, states = [], [], {k: [] for k in STATE_STREAM}
    for _ in range(steps):
        a = torch.as_tensor(policy(obs), dtype=torch.float32, device=env.device)
        r = env.step(a)
        obs = r.obs
        actions.append(a.clone())
        success.append(r.info["success"].clone())
        if store_states:
            for k in STATE_STREAM:
                states[k].append(getattr(env.scene, k).clone())
    cams = getattr(env, "custom_cameras", None)
    manifest = {"engine": __version__, "abi": nat.ABI_VERSION, "task": getattr(env, "task_name", env.name),
                "overrides": getattr(env, "overrides", {}), "num_envs": env.num_envs, "seed": env.seed,
                # everything else make_task and the env were given: the global batch and this shard,
                # the SimConfig, custom cameras and the full step params (eval mode, reset policy ...)
                "global_num_envs": getattr(env, "global_num_envs", env.num_envs),
                "shard": list(env.shard) if getattr(env, "shard", None) else None,
                "env_offset": env.scene.env_offset, "sim": dataclasses.asdict(env.sim),
                "cameras": [dataclasses.asdict(c) for c in cams] if cams else None,
                "c_params": _struct_dict(env.c_params),
                "obs_mode": env.obs_mode, "layout_hash": env.scene.layout_hash,
                "controller": {"mode": env.scene.control.mode, "action_scale": env.scene.control.action_scale},
                "action_dim": env.action_dim, "steps": steps, "source": source, "created": time.time(),
                "initial": {}, "states": {}}
    for k, v in snap0.items():
        if k != "layout_hash":
            manifest["initial"][k] = _write(os.path.join(path, "initial"), k, v.cpu().numpy())
    manifest["actions"] = _write(path, "actions", torch.stack(actions).cpu().numpy() if steps else
                                 np.zeros((0, env.num_envs, env.action_dim), np.float32))
    manifest["success"] = _write(path, "success", torch.stack(success).cpu().numpy() if steps else
                                 np.zeros((0, env.num_envs), np.uint8))
    if store_states and steps:
        for k in STATE_STREAM:
            manifest["states"][k] = _write(os.path.join(path, "states"), k, torch.stack(states[k]).cpu().numpy())
    with open(os.path.join(path, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    return manifest


def _struct_dict(c) -> dict:
    out = {}
    for name, _ in c._fields_:
        v = getattr(c, name)
        out[name] = list(v) if hasattr(v, "__len__") else v
    return out


def _apply_struct(c, d: dict) -> None:
    for name, _ in c._fields_:
        if name not in d:
            continue
        v = d[name]
        if isinstance(v, list):
            arr = getattr(c, name)
            for i, x in enumerate(v):
                arr[i] = x
        else:
            setattr(c, name, v)


def _deviation(got: np.ndarray, rec: np.ndarray) -> float:
    """Max |got - rec|; 0.0 only for a bitwise match (NaNs in the same places count as equal);
    any non-finite difference (NaN vs number, inf - inf) is an infinite deviation."""
    if got.size == 0 or np.array_equal(got, rec, equal_nan=True):
        return 0.0
    d = np.abs(got.astype(np.float64) - rec.astype(np.float64))
    if not np.isfinite(d).all():
        return math.inf
    return float(d.max())


def load(path: str) -> dict:
    with open(os.path.join(path, "manifest.json")) as f:
        man = json.load(f)
    traj = {"manifest": man,
            "initial": {k: _read(os.path.join(path, "initial"), k, m) for k, m in man["initial"].items()},
            "actions": _read(path, "actions", man["actions"]), "success": _read(path, "success", man["success"]),
            "states": {k: _read(os.path.join(path, "states"), k, m) for k, m in man.get("states", {}).items()}}
    return traj


def replay(path: str, obs_mode: str = None, keep_obs: bool = False, device=None):
    """Re-simulate a TrajectoryFile from its initial snapshot with its recorded actions.

    Returns (report, obs_stream).  The report holds, per stored state field, the max
    absolute deviation from the recorded stream (0.0 = bitwise) and whether the success
    flags match.  `obs_mode` regenerates observations (e.g. "rgbd") along the same
    trajectory; `keep_obs` returns them (host copies)."""
    from .tasks import make_task

    traj = load(path)
    man = traj["manifest"]
    if man["engine"] != __version__ or man["abi"] != nat.ABI_VERSION:
        raise LayoutMismatchError(f"trajectory from engine {man['engine']}/ABI {man['abi']}; this is "
                                  f"{__version__}/ABI {nat.ABI_VERSION}")
    from .cameras import CameraConfig
    from .envs import SimConfig

    cams = [CameraConfig(**{k: tuple(v) if isinstance(v, list) else v for k, v in c.items()})
            for c in man["cameras"]] if man.get("cameras") else None
    sim = SimConfig(**{k: tuple(v) if isinstance(v, list) else v for k, v in man["sim"].items()}) \
        if man.get("sim") else None
    shard = tuple(man["shard"]) if man.get("shard") else None
    env = make_task(man["task"], man.get("global_num_envs", man["num_envs"]), seed=man["seed"],
                    overrides=man["overrides"], obs_mode=obs_mode or man["obs_mode"], device=device, shard=shard,
                    sim=sim, cameras=cams)
    if env.num_envs != man["num_envs"] or env.scene.env_offset != man.get("env_offset", 0):
        raise LayoutMismatchError("replayed shard does not match the recorded env range")
    if man.get("c_params"):
        _apply_struct(env.c_params, man["c_params"])  # eval mode, reset policy, seed as recorded
    if env.scene.layout_hash != man["layout_hash"]:
        raise LayoutMismatchError(f"layout {env.scene.layout_hash} != recorded {man['layout_hash']}")
    snap = {k: torch.as_tensor(v, device=env.device) for k, v in traj["initial"].items()}
    snap["layout_hash"] = man["layout_hash"]
    env.scene.set_state(snap)
    if env.renderer is not None:
        env.renderer.render(env.scene)
    dev = {k: 0.0 for k in traj["states"]}
    success_ok = True
    obs_stream = []
    acts = traj["actions"]
    for t in range(len(acts)):
        r = env.step(torch.as_tensor(acts[t], device=env.device))
        if not np.array_equal(r.info["success"].cpu().numpy(), traj["success"][t]):
            success_ok = False
        for k, rec in traj["states"].items():
            dev[k] = max(dev[k], _deviation(getattr(env.scene, k).cpu().numpy(), rec[t]))
        if keep_obs:
            o = r.obs
            obs_stream.append({k: v.cpu().numpy() for k, v in _flat(o).items()} if isinstance(o, dict)
                              else o.cpu().numpy())
    report = {"max_abs_deviation": dev, "bitwise": all(v == 0.0 for v in dev.values()),
              "success_match": success_ok, "steps": len(acts)}
    return report, obs_stream


def _flat(d, prefix=""):
    out = {}
    for k, v in d.items():
        if isinstance(v, dict):
            out.update(_flat(v, prefix + k + "/"))
        else:
            out[prefix + k] = v
    return out
