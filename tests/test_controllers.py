"""Controller surface: action spaces, conversion identities and round trips.
CPU only -- the targets computed here use the same rule the step kernel applies (the GPU
parity tests cover the kernel)."""

import math

import pytest
import torch

from paper_2410_00425_b200.controllers import action_space, convert_action, ee_delta_from_joint_target, joint_targets


def test_action_space_dims():
    assert action_space("pd_joint_pos", 7)["shape"] == (7,)
    assert action_space("pd_ee_delta_pose", 3)["shape"] == (6,)
    assert action_space("base_forward_rotate", 0)["shape"] == (2,)


def test_delta_hold_and_limit_clamp():
    q = torch.tensor([[0.1, -0.2, 0.3]], dtype=torch.float64)
    lo = torch.tensor([-1.0, -1.0, -1.0], dtype=torch.float64)
    hi = torch.tensor([1.0, 1.0, 0.35], dtype=torch.float64)
    assert torch.equal(joint_targets("pd_joint_delta_pos", 0.1, q, lo, hi, torch.zeros(1, 3)), q)  # hold
    t = joint_targets("pd_joint_delta_pos", 0.1, q, lo, hi, torch.ones(1, 3))
    assert t[0, 2] == 0.35  # clamps exactly to the limit


def test_conversions():
    rng = torch.Generator().manual_seed(0)
    q = torch.rand((50, 3), generator=rng, dtype=torch.float64) * 2 - 1
    lo, hi = torch.full((3,), -2.0, dtype=torch.float64), torch.full((3,), 2.0, dtype=torch.float64)
    a = torch.rand((50, 3), generator=rng, dtype=torch.float64) * 2 - 1
    # identity conversion returns the same action
    same, res = convert_action("pd_joint_pos", "pd_joint_pos", q, lo, hi, a)
    assert torch.equal(same, a) and (res == 0).all()
    # joint_pos -> joint_delta_pos: action' = (target - q) / scale; representable ones round-trip
    b, res = convert_action("pd_joint_pos", "pd_joint_delta_pos", q, lo, hi, a * 0.05, scale_to=1.0)
    t_from = joint_targets("pd_joint_pos", 1.0, q, lo, hi, a * 0.05)
    assert torch.allclose(b, (t_from - q).clamp(-1, 1), atol=1e-12)
    ok = res < 1e-12
    assert ok.any()
    assert torch.allclose(joint_targets("pd_joint_delta_pos", 1.0, q, lo, hi, b)[ok], t_from[ok], atol=1e-12)
    # delta -> pos and back
    c, res = convert_action("pd_joint_delta_pos", "pd_joint_pos", q, lo, hi, a)
    assert (res < 1e-12).all()


def test_ee_delta_from_target_pose():
    a = ee_delta_from_joint_target(torch.zeros(1, 3), torch.tensor([[1.0, 0, 0, 0]]),
                                   torch.tensor([[0.005, 0, 0]]), torch.tensor([[math.cos(0.01), 0, 0, math.sin(0.01)]]))
    assert torch.allclose(a, torch.tensor([[0.5, 0, 0, 0, 0, 0.4]], dtype=torch.float64), atol=1e-9)
    with pytest.raises(Exception):
        action_space("teleport", 3)
