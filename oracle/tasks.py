"""Oracle task layer (numpy) -- test infrastructure (oracle/__init__.py).

PickCube-style tabletop (A-17; SPEC.md:613-614 ReachPose/PushCube predicates):
ARM3 on a fixed base + one free cube on the ground plane.  Reset sampling uses the
per-env Philox streams; reward/success/fail/termination/truncation
follow SPEC.md:545-553 and 578-582 (training mode: early termination + auto-reset).

`spec` is the task's configuration record (numbers only, shared with the product);
everything computed from it is restated here.
"""

from __future__ import annotations

import math

import numpy as np

from . import engine as E
from . import se3
from .dynamics import forward_kinematics
from .model import Model
from .philox import reset_uniforms, uniform


class PickCubeOracle:
    """B envs of the PickCube-style scene, stepped by the oracle engine."""

    N_UNIFORMS = 8

    def __init__(self, spec, desc, num_envs, seed, env_offset=0, cfg=None):
        self.spec = spec
        self.model = Model(desc)
        self.cfg = cfg or E.SimConfig()
        self.B = num_envs
        self.seed = seed
        self.env_ids = np.arange(env_offset, env_offset + num_envs, dtype=np.uint64)
        m = self.model
        D = m.D
        self.ee_link = m.link_names.index(f"arm/{spec.ee_link}")
        kp = np.full(D, spec.kp)
        kd = np.full(D, spec.kd)
        self.drv = E.Drives(kp, kd, np.full(D, spec.force_limit), np.zeros((num_envs, D)))
        self.ctrl = type("Ctrl", (), {"mode": spec.control_mode, "dofs": list(range(D)),
                                      "scale": spec.action_scale})()
        self.reset_count = np.zeros(num_envs, np.uint64)
        self.elapsed = np.zeros(num_envs, np.int32)
        self.goal = np.zeros((num_envs, 3))
        self.st = None
        self.reset()

    # ----------------------------------------------------------------- reset
    def _sample(self, idx):
        s = self.spec
        u = reset_uniforms(self.seed, self.env_ids[idx], self.reset_count[idx], self.N_UNIFORMS)
        n = len(idx)
        q = np.empty((n, 3))
        for k in range(3):
            q[:, k] = s.q_rest[k] + uniform(-s.q_noise, s.q_noise, u[:, k])
        cx = uniform(-s.cube_xy, s.cube_xy, u[:, 3])
        cy = uniform(-s.cube_xy, s.cube_xy, u[:, 4])
        yaw = uniform(-math.pi, math.pi, u[:, 5])
        gx = uniform(-s.goal_xy, s.goal_xy, u[:, 6])
        gy = uniform(-s.goal_xy, s.goal_xy, u[:, 7])
        h = 0.5 * yaw
        aq = se3.qnorm(np.stack([np.cos(h), np.zeros(n), np.zeros(n), np.sin(h)], -1))
        ap = np.stack([cx, cy, np.full(n, s.cube_half)], -1)
        goal = np.stack([gx, gy, np.full(n, s.cube_half)], -1)
        return q, ap, aq, goal

    def reset(self, mask=None):
        idx = np.arange(self.B) if mask is None else np.nonzero(mask)[0]
        q, ap, aq, goal = self._sample(idx)
        m = self.model
        if self.st is None:
            self.st = E.State(np.zeros((self.B, m.D)), np.zeros((self.B, m.D)), np.zeros((self.B, m.A, 3)),
                              np.tile([1.0, 0, 0, 0], (self.B, m.A, 1)), np.zeros((self.B, m.A, 3)),
                              np.zeros((self.B, m.A, 3)), np.zeros(self.B, np.uint8))
        st = self.st
        st.q[idx], st.qd[idx] = q, 0.0
        st.ap[idx, 0], st.aq[idx, 0] = ap, aq
        st.av[idx], st.aw[idx] = 0.0, 0.0
        st.diverged[idx] = 0
        self.goal[idx] = goal
        self.elapsed[idx] = 0
        return self.obs()

    # ----------------------------------------------------------------- step
    def link_poses(self):
        return forward_kinematics(self.model, self.st.q)

    def obs(self):
        st = self.st
        LP, _ = self.link_poses()
        ee = LP[:, self.ee_link]
        parts = [st.q, st.qd, ee, st.ap[:, 0], st.aq[:, 0], st.av[:, 0], st.aw[:, 0], self.goal]
        return np.concatenate(parts, -1).astype(np.float32)

    def evaluate(self):
        st = self.st
        LP, _ = self.link_poses()
        ee = LP[:, self.ee_link]
        cube = st.ap[:, 0]
        d_ee = np.sqrt(np.sum((ee - cube) ** 2, -1))
        dg = cube[:, :2] - self.goal[:, :2]
        d_goal = np.sqrt(np.sum(dg * dg, -1))
        success = d_goal < self.spec.success_dist
        fail = (cube[:, 2] < self.spec.fail_z) | (st.diverged != 0)
        reward = (-(d_ee + d_goal)).astype(np.float32)
        return reward, success, fail

    def step(self, action, want_contacts=False):
        self.st = E.control_step(self.model, self.st, self.drv, self.ctrl, action, self.cfg, want_contacts)
        unsupported = self.st.unsupported
        reward, success, fail = self.evaluate()
        self.elapsed += 1
        terminated = success | fail
        truncated = self.elapsed >= self.spec.max_steps
        info = {"success": success, "fail": fail, "unsupported_pairs": unsupported,
                "diverged": self.st.diverged.copy(), "contacts": self.st.contacts}
        done = terminated | truncated
        final = self.snapshot()
        if done.any():
            self.reset_count[done] += 1
            self.reset(done)
        return self.obs(), reward, terminated, truncated, info, final

    def snapshot(self):
        st = self.st
        return {"q": st.q.copy(), "qd": st.qd.copy(), "ap": st.ap.copy(), "aq": st.aq.copy(),
                "av": st.av.copy(), "aw": st.aw.copy(), "goal": self.goal.copy(), "elapsed": self.elapsed.copy()}

    def load(self, snap):
        st = self.st
        st.q[:], st.qd[:], st.ap[:], st.aq[:] = snap["q"], snap["qd"], snap["ap"], snap["aq"]
        st.av[:], st.aw[:] = snap["av"], snap["aw"]
        self.goal[:] = snap["goal"]
        self.elapsed[:] = snap["elapsed"]
