"""Controller presets, action spaces and action conversion.

The controllers themselves run inside the fused step kernel: they clip the normalised action
and turn it into drive targets (``csrc/step.cu`` "controller"). This module is the host-side
surface:

- ``action_space(mode, n_joints)``: dimension and bounds;
- ``convert_action(cfg_from, cfg_to, qpos, lower, upper, action)``: the algebraic conversions
  between joint-space modes. The EE-delta target of a joint target (FK of
  the target configuration) is handled by ``ee_delta_from_joint_target``;
- the preset table.
"""

from __future__ import annotations

import math

import torch

from .errors import InputError

MODES = ("pd_joint_pos", "pd_joint_delta_pos", "pd_ee_delta_pose", "base_forward_rotate")

PRESETS = {
    "pd_joint_pos": {"action_scale": 1.0},
    "pd_joint_delta_pos": {"action_scale": 0.1},            # rad per unit action (A-22)
    "pd_ee_delta_pose": {"action_scale": 0.01, "action_scale_rot": 0.05, "ik_lambda": 0.05},
}


def action_space(mode: str, n_joints: int) -> dict:
    """[-1, 1]^D box: D = controlled joints (joint modes), 6 (EE delta: xyz + axis-angle),
    or 2 (base: forward, rotate)."""
    if mode not in MODES:
        raise InputError(f"unknown controller mode {mode!r}; one of {MODES}")
    d = {"pd_ee_delta_pose": 6, "base_forward_rotate": 2}.get(mode, n_joints)
    return {"low": -torch.ones(d), "high": torch.ones(d), "shape": (d,)}


def joint_targets(mode: str, scale: float, qpos, lower, upper, action):
    """The kernel's joint-mode target rule, for conversion and tests."""
    a = torch.clamp(torch.as_tensor(action, dtype=torch.float64), -1.0, 1.0)
    q = torch.as_tensor(qpos, dtype=torch.float64)
    lo = torch.as_tensor(lower, dtype=torch.float64)
    hi = torch.as_tensor(upper, dtype=torch.float64)
    if mode == "pd_joint_delta_pos":
        return torch.minimum(torch.maximum(q + a * scale, lo), hi)
    if mode == "pd_joint_pos":
        finite = torch.isfinite(lo) & torch.isfinite(hi)
        un = torch.where(finite, lo + (a + 1.0) * 0.5 * (hi - lo), a * scale)
        return torch.minimum(torch.maximum(un, lo), hi)
    raise InputError(f"{mode} has no joint-target rule")


def convert_action(mode_from: str, mode_to: str, qpos, lower, upper, action, scale_from: float = None,
                   scale_to: float = None):
    """Action under `mode_to` whose drive targets best match `mode_from`'s.

    Returns (action', residual): residual = max |target_to - target_from| after clipping to
    [-1, 1] (non-zero when the target is not representable, reported rather than hidden)."""
    scale_from = PRESETS.get(mode_from, {}).get("action_scale", 1.0) if scale_from is None else scale_from
    scale_to = PRESETS.get(mode_to, {}).get("action_scale", 1.0) if scale_to is None else scale_to
    if mode_from == mode_to and scale_from == scale_to:
        a = torch.as_tensor(action, dtype=torch.float64)
        return a.clone(), torch.zeros(a.shape[:-1], dtype=torch.float64)
    target = joint_targets(mode_from, scale_from, qpos, lower, upper, action)
    q = torch.as_tensor(qpos, dtype=torch.float64)
    lo = torch.as_tensor(lower, dtype=torch.float64)
    hi = torch.as_tensor(upper, dtype=torch.float64)
    if mode_to == "pd_joint_delta_pos":
        out = (target - q) / scale_to
    elif mode_to == "pd_joint_pos":
        finite = torch.isfinite(lo) & torch.isfinite(hi)
        out = torch.where(finite, 2.0 * (target - lo) / torch.where(finite, hi - lo, 1.0) - 1.0, target / scale_to)
    else:
        raise InputError(f"conversion {mode_from} -> {mode_to} is not a joint-space conversion")
    out = torch.clamp(out, -1.0, 1.0)
    back = joint_targets(mode_to, scale_to, q, lo, hi, out)
    return out, (back - target).abs().amax(-1)


def ee_delta_from_joint_target(p_now, q_now, p_target, q_target, scale: float = 0.01, rot_scale: float = 0.05):
    """EE-delta action (xyz + axis-angle, world frame) from the current and the target EE poses
    (FK of the joint target), inverting the action scaling; clipped to [-1, 1]."""
    p_now, p_target = torch.as_tensor(p_now, dtype=torch.float64), torch.as_tensor(p_target, dtype=torch.float64)
    qa, qb = torch.as_tensor(q_now, dtype=torch.float64), torch.as_tensor(q_target, dtype=torch.float64)
    # relative rotation R_target R_now^T as a quaternion: q_t * conj(q_n)
    w1, x1, y1, z1 = qb.unbind(-1)
    w2, x2, y2, z2 = (qa * torch.tensor([1.0, -1.0, -1.0, -1.0], dtype=torch.float64)).unbind(-1)
    dq = torch.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                      w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], -1)
    dq = torch.where(dq[..., :1] < 0, -dq, dq)
    s = dq[..., 1:].norm(dim=-1, keepdim=True)
    ang = 2.0 * torch.atan2(s, dq[..., :1])
    axis = torch.where(s > 1e-12, dq[..., 1:] / s.clamp_min(1e-300), torch.zeros_like(dq[..., 1:]))
    a = torch.cat([(p_target - p_now) / scale, axis * ang / rot_scale], -1)
    return torch.clamp(a, -1.0, 1.0)


def hold_action(mode: str, n: int, d: int) -> torch.Tensor:
    """The zero ("hold") action of a delta controller."""
    if mode not in ("pd_joint_delta_pos", "pd_ee_delta_pose"):
        raise InputError("hold is defined for delta controllers")
    return torch.zeros((n, d))


__all__ = ["MODES", "PRESETS", "action_space", "joint_targets", "convert_action", "ee_delta_from_joint_target",
           "hold_action", "math"]
