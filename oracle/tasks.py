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


def rest_pose(kind, size):
    """DESIGN.md A-26: resting height and orientation of a free primitive on the plane --
    upright box / sphere at half-height / radius; capsule / cylinder lying along world x."""
    if kind in ("box",):
        return float(size[2]), np.array([1.0, 0.0, 0.0, 0.0])
    if kind == "sphere":
        return float(size[0]), np.array([1.0, 0.0, 0.0, 0.0])
    h = math.sqrt(0.5)
    return float(size[0]), np.array([h, 0.0, h, 0.0])


class PickCubeOracle:
    """B envs of the PickCube-style scene, stepped by the oracle engine."""

    N_UNIFORMS = 8

    def __init__(self, spec, desc, num_envs, seed, env_offset=0, cfg=None, env_ids=None):
        self.spec = spec
        self.model = Model(desc)
        self.cfg = cfg or E.SimConfig()
        self.B = num_envs
        self.seed = seed
        self.env_ids = (np.arange(env_offset, env_offset + num_envs, dtype=np.uint64) if env_ids is None
                        else np.asarray(env_ids, np.uint64))
        self.rest_z, self.rest_q = rest_pose(desc.actors[0].kind, desc.actors[0].size)
        m = self.model
        D = m.D
        self.ee_link = m.link_names.index(f"arm/{spec.ee_link}")
        kp = np.full(D, spec.kp)
        kd = np.full(D, spec.kd)
        self.drv = E.Drives(kp, kd, np.full(D, spec.force_limit), np.zeros((num_envs, D)))
        self.ctrl = type("Ctrl", (), {"mode": spec.control_mode, "dofs": list(range(D)),
                                      "scale": spec.action_scale, "rot_scale": 0.05, "lam": 0.05,
                                      "ee_link": self.ee_link})()
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
        if tuple(self.rest_q) != (1.0, 0.0, 0.0, 0.0):
            aq = se3.qnorm(se3.qmul(aq, np.broadcast_to(self.rest_q, aq.shape)))
        ap = np.stack([cx, cy, np.full(n, self.rest_z)], -1)
        goal = np.stack([gx, gy, np.full(n, self.rest_z)], -1)
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


class OpenCabinetOracle:
    """Heterogeneous OpenCabinet (OpenChain-Hetero; A-18): envs are grouped
    by layout and each group is stepped by the oracle engine (envs are independent,
    SPEC.md:216).  Reset: arm at q_rest + U(-noise, noise); cabinet parts closed; target part
    = 3 + floor(u3 * n_parts).  success = q_target > frac * upper; reward = q_target / upper."""

    N_UNIFORMS = 8

    def __init__(self, spec, descs, seed, env_offset=0, cfg=None):
        self.spec = spec
        self.cfg = cfg or E.SimConfig()
        self.B = len(descs)
        self.seed = seed
        self.env_ids = np.arange(env_offset, env_offset + self.B, dtype=np.uint64)
        groups = {}
        for e, d in enumerate(descs):
            groups.setdefault(d.key(), (d, []))[1].append(e)
        self.groups = []
        for d, idx in groups.values():
            m = Model(d)
            D = m.D
            kp = np.zeros(D)
            kd = np.zeros(D)
            fl = np.full(D, np.inf)
            kp[:3], kd[:3], fl[:3] = spec.kp, spec.kd, spec.force_limit
            drv = E.Drives(kp, kd, fl, np.zeros((len(idx), D)))
            ctrl = type("Ctrl", (), {"mode": spec.control_mode, "dofs": [0, 1, 2], "scale": spec.action_scale})()
            self.groups.append({"model": m, "idx": np.asarray(idx), "drv": drv, "ctrl": ctrl, "st": None,
                                "ee": m.link_names.index(f"arm/{spec.ee_link}")})
        self.D_max = max(g["model"].D for g in self.groups)
        self.reset_count = np.zeros(self.B, np.uint64)
        self.elapsed = np.zeros(self.B, np.int32)
        self.target = np.full(self.B, -1, np.int64)
        self.reset()

    def reset(self, mask=None):
        s = self.spec
        for g in self.groups:
            m, idx = g["model"], g["idx"]
            sel = np.arange(len(idx)) if mask is None else np.nonzero(mask[idx])[0]
            if g["st"] is None:
                B = len(idx)
                g["st"] = E.State(np.zeros((B, m.D)), np.zeros((B, m.D)), np.zeros((B, 0, 3)),
                                  np.zeros((B, 0, 4)), np.zeros((B, 0, 3)), np.zeros((B, 0, 3)), np.zeros(B, np.uint8))
            if not len(sel):
                continue
            ge = idx[sel]
            u = reset_uniforms(self.seed, self.env_ids[ge], self.reset_count[ge], self.N_UNIFORMS)
            st = g["st"]
            st.q[sel] = 0.0
            st.qd[sel] = 0.0
            for k in range(3):
                st.q[sel, k] = s.q_rest[k] + uniform(-s.q_noise, s.q_noise, u[:, k])
            nobj = m.D - 3
            self.target[ge] = 3 + np.minimum((u[:, 3] * nobj).astype(np.int64), nobj - 1) if nobj > 0 else -1
            st.diverged[sel] = 0
            self.elapsed[ge] = 0

    def step(self, action):
        action = np.asarray(action)
        reward = np.zeros(self.B, np.float32)
        success = np.zeros(self.B, bool)
        fail = np.zeros(self.B, bool)
        for g in self.groups:
            m, idx = g["model"], g["idx"]
            g["st"] = E.control_step(m, g["st"], g["drv"], g["ctrl"], action[idx], self.cfg)
            t = self.target[idx]
            rows = np.arange(len(idx))
            hi = m.upper[t]
            qv = g["st"].q[rows, t]
            success[idx] = qv > self.spec.success_frac * hi
            reward[idx] = (qv / hi).astype(np.float32)
            fail[idx] = g["st"].diverged != 0
        self.elapsed += 1
        terminated = success | fail
        truncated = self.elapsed >= self.spec.max_steps
        info = {"success": success, "fail": fail}
        done = terminated | truncated
        final = self.snapshot()
        if done.any():
            self.reset_count[done] += 1
            self.reset(done)
        return reward, terminated, truncated, info, final

    def snapshot(self):
        q = np.zeros((self.B, self.D_max))
        qd = np.zeros((self.B, self.D_max))
        ee = np.zeros((self.B, 3))
        for g in self.groups:
            m, idx = g["model"], g["idx"]
            q[idx, :m.D] = g["st"].q
            qd[idx, :m.D] = g["st"].qd
            LP, _ = forward_kinematics(m, g["st"].q)
            ee[idx] = LP[:, g["ee"]]
        return {"q": q, "qd": qd, "ee": ee, "target": self.target.copy(), "elapsed": self.elapsed.copy()}

    def load(self, q, qd):
        for g in self.groups:
            m, idx = g["model"], g["idx"]
            g["st"].q[:] = q[idx, :m.D]
            g["st"].qd[:] = qd[idx, :m.D]


class PickHeteroOracle:
    """PickHetero (BASELINE config 5): envs grouped by object layout, each group a
    PickCubeOracle over its global env ids (envs are independent)."""

    def __init__(self, spec, descs, seed, cfg=None, env_offset=0):
        self.B = len(descs)
        groups = {}
        for e, d in enumerate(descs):
            groups.setdefault(d.key(), (d, []))[1].append(e)
        self.groups = [(np.asarray(idx), PickCubeOracle(spec, d, len(idx), seed, cfg=cfg,
                                                        env_ids=np.asarray(idx) + env_offset))
                       for d, idx in groups.values()]

    def step(self, action):
        rew = np.zeros(self.B, np.float32)
        term = np.zeros(self.B, bool)
        trunc = np.zeros(self.B, bool)
        succ = np.zeros(self.B, bool)
        for idx, o in self.groups:
            _, r, te, tr, info, _ = o.step(np.asarray(action)[idx])
            rew[idx], term[idx], trunc[idx], succ[idx] = r, te, tr, info["success"]
        return rew, term, trunc, {"success": succ}

    def snapshot(self):
        out = {}
        for idx, o in self.groups:
            sn = o.snapshot()
            for k, v in sn.items():
                if k not in out:
                    out[k] = np.zeros((self.B,) + v.shape[1:], v.dtype)
                out[k][idx] = v
        return out

    def load(self, snap, reset_count=None):
        for idx, o in self.groups:
            o.load({k: v[idx] for k, v in snap.items()})
            if reset_count is not None:
                o.reset_count[:] = reset_count[idx]

    def link_poses(self):
        return [(idx, o.link_poses(), o) for idx, o in self.groups]


class CartpoleOracle:
    """CartpoleBalance (A-27): the cartpole fixture, slider driven by
    pd_joint_delta_pos, hinge passive.  Reset: slider, hinge and both rates ~ U(-noise, noise)
    from reset uniforms 0..3.  Per control step: streak = streak + 1 if |theta| < success_angle
    else 0; success = streak >= success_steps; fail = |theta| > fail_angle or |x| > fail_x or
    diverged; reward = cos(theta) (float32); obs = (x, x_dot, theta, theta_dot)."""

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
        slider = 0  # fixture order: dof 0 = slider (cart), dof 1 = hinge (pole)
        kp, kd, fl = np.zeros(D), np.zeros(D), np.full(D, np.inf)
        kp[slider], kd[slider], fl[slider] = spec.kp, spec.kd, spec.force_limit
        self.drv = E.Drives(kp, kd, fl, np.zeros((num_envs, D)))
        self.ctrl = type("Ctrl", (), {"mode": spec.control_mode, "dofs": [slider], "scale": spec.action_scale})()
        self.reset_count = np.zeros(num_envs, np.uint64)
        self.elapsed = np.zeros(num_envs, np.int32)
        self.streak = np.zeros(num_envs, np.int32)
        self.st = None
        self.reset()

    def reset(self, mask=None):
        idx = np.arange(self.B) if mask is None else np.nonzero(mask)[0]
        m = self.model
        if self.st is None:
            self.st = E.State(np.zeros((self.B, m.D)), np.zeros((self.B, m.D)), np.zeros((self.B, 0, 3)),
                              np.zeros((self.B, 0, 4)), np.zeros((self.B, 0, 3)), np.zeros((self.B, 0, 3)),
                              np.zeros(self.B, np.uint8))
        if len(idx):
            u = reset_uniforms(self.seed, self.env_ids[idx], self.reset_count[idx], self.N_UNIFORMS)
            n = self.spec.init_noise
            st = self.st
            for i in range(2):
                st.q[idx, i] = uniform(-n, n, u[:, i])
                st.qd[idx, i] = uniform(-n, n, u[:, 2 + i])
            st.diverged[idx] = 0
            self.elapsed[idx] = 0
            self.streak[idx] = 0
        return self.obs()

    def obs(self):
        q, qd = self.st.q, self.st.qd
        return np.stack([q[:, 0], qd[:, 0], q[:, 1], qd[:, 1]], -1).astype(np.float32)

    def step(self, action):
        s = self.spec
        self.st = E.control_step(self.model, self.st, self.drv, self.ctrl, np.asarray(action), self.cfg)
        x, th = self.st.q[:, 0], self.st.q[:, 1]
        self.streak = np.where(np.abs(th) < s.success_angle, self.streak + 1, 0).astype(np.int32)
        success = self.streak >= s.success_steps
        fail = (np.abs(th) > s.fail_angle) | (np.abs(x) > s.fail_x) | (self.st.diverged != 0)
        reward = np.cos(th).astype(np.float32)
        self.elapsed += 1
        terminated = success | fail
        truncated = self.elapsed >= s.max_steps
        info = {"success": success, "fail": fail}
        done = terminated | truncated
        final = {"q": self.st.q.copy(), "qd": self.st.qd.copy(), "streak": self.streak.copy(),
                 "elapsed": self.elapsed.copy()}
        if done.any():
            self.reset_count[done] += 1
            self.reset(done)
        return self.obs(), reward, terminated, truncated, info, final
