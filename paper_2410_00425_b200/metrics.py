"""Episode metrics, the evaluation wrapper and keyed action maps.

- EpisodeMetrics are accumulated inside the fused step kernel, per env, for every episode
  (return = sum of rewards, length, success_once / success_at_end, fail_once /
  fail_at_end). When an episode ends, the kernel writes its record to the env's ``ep_*``
  output buffers and flags ``ep_done``. Nothing here adds a launch to the step.
- ``EpisodeStats`` sums the finished episodes on the device (a handful of tiny reductions,
  run when the caller asks). ``paper_2410_00425_b200.dist.reduce_stats`` all-reduces them
  across ranks at rollout boundaries.
- ``MetricsSink`` writes one JSON line per finished episode with exactly the SPEC's fields
  (return, length, success_once, success_at_end, fail_once, fail_at_end, env_id, seed). It
  copies to the host, so call it only when logging.
- ``eval_wrapper`` turns off early termination and auto-reset. Episodes then
  always run to the time limit and metrics are emitted at truncation.
- ``flatten_action_map`` / ``unflatten_action`` handle keyed multi-agent actions in sorted
  agent order.
"""

from __future__ import annotations

import json

import torch

from .dist import STAT_FIELDS
from .errors import InputError

FLAG_SUCCESS_ONCE, FLAG_SUCCESS_AT_END, FLAG_FAIL_ONCE, FLAG_FAIL_AT_END = 1, 2, 4, 8


def episode_records(info) -> dict:
    """Device tensors describing the episodes that ended in the last step (mask + fields)."""
    ep = info["episode"]
    f = ep["flags"]
    return {"done": ep["done"].bool(), "return": ep["return"], "length": ep["length"],
            "success_once": (f & FLAG_SUCCESS_ONCE) != 0, "success_at_end": (f & FLAG_SUCCESS_AT_END) != 0,
            "fail_once": (f & FLAG_FAIL_ONCE) != 0, "fail_at_end": (f & FLAG_FAIL_AT_END) != 0}


class EpisodeStats:
    """Device-side running sums over finished episodes, in dist.STAT_FIELDS order."""

    def __init__(self, device):
        self.sums = torch.zeros(len(STAT_FIELDS), dtype=torch.float64, device=device)

    def update(self, info) -> None:
        r = episode_records(info)
        d = r["done"]
        df = d.double()
        self.sums += torch.stack([df.sum(), (r["return"] * df).sum(), (r["length"].double() * df).sum(),
                                  (r["success_once"] & d).double().sum(), (r["success_at_end"] & d).double().sum(),
                                  (r["fail_once"] & d).double().sum(), (r["fail_at_end"] & d).double().sum()])

    def reset(self) -> None:
        self.sums.zero_()


class MetricsSink:
    """JSON-lines sink of finished episodes."""

    FIELDS = ("return", "length", "success_once", "success_at_end", "fail_once", "fail_at_end", "env_id", "seed")

    def __init__(self, path: str, seed: int, env_offset: int = 0):
        self.path, self.seed, self.env_offset = path, int(seed), int(env_offset)
        self._f = open(path, "a")
        self.count = 0

    def write(self, info) -> int:
        r = episode_records(info)
        done = r["done"].cpu()
        idx = torch.nonzero(done).flatten().tolist()
        if not idx:
            return 0
        cols = {k: r[k].cpu() for k in ("return", "length", "success_once", "success_at_end", "fail_once",
                                         "fail_at_end")}
        for i in idx:
            rec = {"return": float(cols["return"][i]), "length": int(cols["length"][i]),
                   "success_once": bool(cols["success_once"][i]), "success_at_end": bool(cols["success_at_end"][i]),
                   "fail_once": bool(cols["fail_once"][i]), "fail_at_end": bool(cols["fail_at_end"][i]),
                   "env_id": self.env_offset + i, "seed": self.seed}
            self._f.write(json.dumps(rec) + "\n")
        self._f.flush()
        self.count += len(idx)
        return len(idx)

    def close(self) -> None:
        self._f.close()


def eval_wrapper(env):
    """Evaluation mode: terminated is never raised early and envs are not
    auto-reset, so every episode runs to its time limit; metrics are emitted at truncation.
    Mutates and returns `env`; captured CUDA graphs (device and host-I/O) are re-captured on
    their next replay because the params they baked in changed (envs.Env._replay)."""
    env.c_params.early_termination = 0
    env.c_params.auto_reset = 0
    env.eval_mode = True
    return env


def flatten_action_map(keyed: dict, dims: dict) -> torch.Tensor:
    """Concatenate per-agent actions in sorted agent order."""
    missing = sorted(set(dims) - set(keyed))
    unknown = sorted(set(keyed) - set(dims))
    if missing or unknown:
        raise InputError(f"action map mismatch: missing {missing}, unknown {unknown}")
    parts = []
    for name in sorted(dims):
        a = torch.as_tensor(keyed[name])
        if a.shape[-1] != dims[name]:
            raise InputError(f"agent {name!r}: action dim {a.shape[-1]} != {dims[name]}")
        parts.append(a)
    return torch.cat(parts, dim=-1) if len(parts) > 1 else parts[0]


def unflatten_action(flat: torch.Tensor, dims: dict) -> dict:
    """Inverse of flatten_action_map (exact slices)."""
    out, k = {}, 0
    for name in sorted(dims):
        out[name] = flat[..., k:k + dims[name]]
        k += dims[name]
    if k != flat.shape[-1]:
        raise InputError(f"flat action has dim {flat.shape[-1]}, agents need {k}")
    return out
