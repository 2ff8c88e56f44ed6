"""Vectorised environment protocol over the device scene store.

``Env.step(action)`` is one fused kernel launch (``bs_step``: controller -> substeps ->
FK -> task evaluation -> state obs -> in-kernel auto-reset), followed by one render launch
when the obs mode has cameras.  With ``use_graph=True`` the whole sequence is captured
once into a CUDA graph and replayed, so a step costs one graph launch of host time.

Results are device tensors; nothing is copied to the host unless the caller asks.  With
graphs enabled the returned tensors are the env's static output buffers (overwritten by
the next step) -- clone them to keep a history.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _native as nat
from . import cabi
from .errors import BS_ERR_INPUT, DimensionError, InputError, raise_for_status


@dataclass
class SimConfig:
    """SPEC.md:306 with the Appendix-B names; defaults = the paper's benchmark setup
    (PAPER.md:386-394): sim 120 Hz, control 60 Hz, 4 position / 0 velocity iterations."""

    sim_freq: int = 120
    control_freq: int = 60
    solver_pos_iters: int = 4
    solver_vel_iters: int = 0
    gravity: tuple = (0.0, 0.0, -9.81)
    friction_coeff: float = 1.0
    restitution: float = 0.0
    penetration_slop: float = 5e-4
    baumgarte_beta: float = 0.2

    def __post_init__(self):
        if self.sim_freq % self.control_freq:
            raise ValueError("sim_freq must be divisible by control_freq")
        if self.solver_pos_iters < 0 or self.solver_vel_iters < 0:
            raise ValueError("solver iterations must be >= 0")


class StepResult(NamedTuple):
    obs: object
    reward: torch.Tensor
    terminated: torch.Tensor
    truncated: torch.Tensor
    info: dict


class Env:
    """N parallel envs of one task on one GPU (one shard of a multi-GPU batch)."""

    def __init__(self, scene, task: int, task_f, ee_link: int, max_steps: int, seed: int,
                 sim: SimConfig = None, obs_mode: str = "state", renderer=None, auto_reset: bool = True,
                 early_termination: bool = True, validate_actions: bool = True, name: str = "task"):
        self.scene = scene
        self.name = name
        self.sim = sim or SimConfig()
        self.num_envs = scene.num_envs
        self.device = scene.device
        self.obs_mode = obs_mode
        self.renderer = renderer
        self.validate_actions = validate_actions
        self.action_dim = scene.action_dim
        self.seed = int(seed)
        ctl = scene.control
        p = cabi.BsSimParams()
        p.dt = 1.0 / self.sim.sim_freq
        p.substeps = self.sim.sim_freq // self.sim.control_freq
        p.control_freq = float(self.sim.control_freq)
        p.pos_iters, p.vel_iters = self.sim.solver_pos_iters, self.sim.solver_vel_iters
        for i in range(3):
            p.gravity[i] = self.sim.gravity[i]
        p.friction, p.beta, p.slop = self.sim.friction_coeff, self.sim.baumgarte_beta, self.sim.penetration_slop
        p.ctrl_mode = cabi.CTRL[ctl.mode]
        p.action_dim = self.action_dim
        p.action_scale, p.ik_lambda = ctl.action_scale, ctl.ik_lambda
        p.action_scale_rot = getattr(ctl, "action_scale_rot", 0.05)
        p.ee_link, p.task, p.max_steps = ee_link, task, max_steps
        p.auto_reset, p.early_termination = int(auto_reset), int(early_termination)
        p.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        for i, v in enumerate(task_f):
            p.task_f[i] = v
        self.c_params = p
        N, dev = self.num_envs, self.device
        # state obs layout; CartpoleBalance: (x, x_dot, theta, theta_dot)
        self.obs_dim = 4 if task == cabi.TASK_CARTPOLE else 2 * scene.D_max + 3 + 13 * scene.A_max + 3
        # the per-step host-facing outputs (state obs, reward, four flag bytes) are views of ONE
        # contiguous device arena, so the host-I/O path reads them back with a single copy
        self._arena_layout = [("obs", (N, self.obs_dim), torch.float32), ("reward", (N,), torch.float32),
                              ("terminated", (N,), torch.uint8), ("truncated", (N,), torch.uint8),
                              ("success", (N,), torch.uint8), ("fail", (N,), torch.uint8)]
        self._out_arena = torch.zeros(self._arena_bytes(), dtype=torch.uint8, device=dev)
        v = self._arena_views(self._out_arena)
        self.state_obs, self.reward = v["obs"], v["reward"]
        self.terminated, self.truncated, self.success, self.fail = (v["terminated"], v["truncated"], v["success"],
                                                                    v["fail"])
        self.unsupported = torch.zeros(N, dtype=torch.int32, device=dev)
        self.contact_count = torch.zeros(N, dtype=torch.int32, device=dev)
        self.contact_pairs = torch.zeros((N, scene.C_max, 2), dtype=torch.int32, device=dev)
        self.contact_geom = torch.zeros((N, scene.C_max, 7), dtype=torch.float64, device=dev)
        self.action_buf = torch.zeros((N, max(1, self.action_dim)), dtype=torch.float32, device=dev)
        self.ep_done = torch.zeros(N, dtype=torch.uint8, device=dev)
        self.ep_return_out = torch.zeros(N, dtype=torch.float64, device=dev)
        self.ep_length_out = torch.zeros(N, dtype=torch.int32, device=dev)
        self.ep_flags_out = torch.zeros(N, dtype=torch.uint8, device=dev)
        # state obs of the state an episode ended in (written for auto-reset envs only)
        self.final_obs = torch.zeros((N, self.obs_dim), dtype=torch.float32, device=dev)
        o = cabi.BsStepOutputs()
        o.obs, o.obs_dim = self.state_obs.data_ptr(), self.obs_dim
        for k, t in (("reward", self.reward), ("terminated", self.terminated), ("truncated", self.truncated),
                     ("success", self.success), ("fail", self.fail), ("unsupported_pairs", self.unsupported),
                     ("contact_count", self.contact_count), ("contact_pairs", self.contact_pairs),
                     ("contact_geom", self.contact_geom), ("ep_done", self.ep_done),
                     ("ep_return_out", self.ep_return_out), ("ep_length_out", self.ep_length_out),
                     ("ep_flags_out", self.ep_flags_out), ("final_obs", self.final_obs)):
            setattr(o, k, t.data_ptr())
        self.c_out = o
        self._graph = None
        self._graph_key = None
        self._host_graph = None
        self._host_graph_key = None
        self._warmed = False

    # ------------------------------------------------------------------ spaces
    @property
    def action_space(self):
        """Box [-1, 1]^D_c."""
        lo = -torch.ones(self.action_dim)
        return {"low": lo, "high": -lo, "shape": (self.action_dim,)}

    # ------------------------------------------------------------------ protocol
    def reset(self, seed=None, env_mask=None):
        """Re-initialise the selected envs from their RNG streams.
        A new `seed` re-keys every env's stream; the mask selects a partial reset."""
        if seed is not None:
            self.seed = int(seed)
            self.c_params.seed = self.seed & 0xFFFFFFFFFFFFFFFF
            self.scene.reset_count.zero_()
            bump = 0
        else:
            bump = 1 if env_mask is not None else 0
        mask = None
        if env_mask is not None:
            mask = torch.as_tensor(env_mask, device=self.device).to(torch.uint8).contiguous()
            if mask.shape != (self.num_envs,):
                raise DimensionError(f"env_mask must have shape ({self.num_envs},)")
        nat.call("bs_reset", ctypes.byref(self.scene.c_tables), ctypes.byref(self.scene.c_state),
                 ctypes.byref(self.c_out), ctypes.byref(self.c_params),
                 None if mask is None else mask.data_ptr(), bump, nat.stream_handle())
        self._render()
        return self._obs()

    def _launch_sim(self, action_ptr):
        nat.call("bs_step", ctypes.byref(self.scene.c_tables), ctypes.byref(self.scene.c_state),
                 ctypes.byref(self.c_out), ctypes.byref(self.c_params), action_ptr, nat.stream_handle())

    def _launch_step(self, action_ptr):
        self._launch_sim(action_ptr)
        self._render()

    def _render(self):
        if self.renderer is not None:
            self.renderer.render(self.scene)

    def step(self, action) -> StepResult:
        """controller -> dynamics -> task evaluation -> reward.

        `action` may live on the host (numpy / CPU tensor; validated there and copied
        asynchronously, from pinned memory when the caller provides it) or on the device
        (validated with one device reduction, which synchronises; pass
        validate_actions=False to the env to skip it)."""
        a = action if isinstance(action, torch.Tensor) else torch.as_tensor(action)
        if a.shape != (self.num_envs, self.action_dim):
            raise DimensionError(f"action must have shape ({self.num_envs}, {self.action_dim}), "
                                 f"got {tuple(a.shape)}")
        if self.validate_actions:
            finite = torch.isfinite(a).all()
            if not bool(finite):
                raise InputError("non-finite action")
        if a.numel() == 0:  # no controlled dofs (e.g. a scene of free bodies): any valid buffer
            ptr = self.action_buf.data_ptr()
        elif a.device != self.device or a.dtype != torch.float32 or not a.is_contiguous():
            self.action_buf.copy_(a, non_blocking=True)
            ptr = self.action_buf.data_ptr()
        elif self._graph is not None:
            self.action_buf.copy_(a)
            ptr = self.action_buf.data_ptr()
        else:
            ptr = a.data_ptr()
        if self._graph is not None:
            self._replay()
        else:
            self._launch_step(ptr)
        return self._result()

    def random_actions(self, step_index: int) -> torch.Tensor:
        """Philox uniform actions in [-1, 1) for every env, generated on the device into the
        static action buffer (the benchmark's random-action stream)."""
        nat.call("bs_random_actions", self.seed, step_index, self.scene.env_offset, self.num_envs,
                 self.action_dim, self.action_buf.data_ptr(), nat.stream_handle())
        return self.action_buf

    def launch_step(self) -> None:
        """Enqueue one step on the static action buffer (no validation, no host work)."""
        if self._graph is not None:
            self._replay()
        else:
            self._launch_step(self.action_buf.data_ptr())

    def step_random(self, step_index: int) -> StepResult:
        """Benchmark helper: Philox random actions generated on the device, then step."""
        self.random_actions(step_index)
        self.launch_step()
        return self._result()

    # ------------------------------------------------------------------ CUDA graphs
    # A graph bakes in the BsSimParams it was captured with (bs_step takes them by value into
    # the kernel's constant bank).  Every graph records the params bytes it was captured
    # with; a step whose params differ (reset(seed=...), eval_wrapper, a user edit) re-captures
    # before replaying, so a graph never replays stale seeds or reset/termination modes.

    def _params_key(self) -> bytes:
        return bytes(self.c_params)

    def _side_effect_buffers(self):
        """Every device buffer a step writes outside the scene state rows."""
        bufs = [self._out_arena, self.unsupported, self.contact_count, self.contact_pairs, self.contact_geom,
                self.ep_done, self.ep_return_out, self.ep_length_out, self.ep_flags_out, self.final_obs]
        if self.renderer is not None:
            for g in self.renderer.groups:
                bufs += [g[k] for k in ("rgb", "depth", "seg", "pc") if g[k] is not None]
        return bufs

    def _warm_launchers(self, launch) -> None:
        """Run `launch` once eagerly so every launcher has configured its kernels (shared-memory
        opt-in, occupancy queries) before a capture, then restore EVERYTHING it wrote: the
        scene state and every output buffer -- the warmup leaves no trace."""
        if self._warmed:
            return
        cur = torch.cuda.current_stream(self.device)
        snap = self.scene.get_state()                      # queued on the current stream first
        saved = [b.clone() for b in self._side_effect_buffers()]
        launch()                                           # same stream: ordered after the snapshot
        self.scene.set_state(snap)
        for b, v in zip(self._side_effect_buffers(), saved):
            b.copy_(v)
        cur.synchronize()
        self._warmed = True

    def _capture(self, launch) -> "torch.cuda.CUDAGraph":
        self._warm_launchers(launch)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):   # capture records, it does not execute: no state changes
            launch()
        return g

    def capture_graph(self) -> None:
        """Capture bs_step (+ render) on the static action buffer into a CUDA graph (after one
        side-effect-free eager warm-up of the launchers the first time)."""
        self._graph = self._capture(lambda: self._launch_step(self.action_buf.data_ptr()))
        self._graph_key = self._params_key()

    def _replay(self) -> None:
        if self._graph_key != self._params_key():
            self.capture_graph()
        self._graph.replay()

    # ------------------------------------------------------------------ host I/O path
    def enable_host_io(self) -> None:
        """Capture [step reading the host actions and writing obs/reward/flags to host memory
        (zero-copy over PCIe), render, D2H of the frames] as ONE CUDA graph over pinned host
        buffers, for callers that keep actions and observations on the host (``step_host``).
        The device-side API (``step``) is unaffected; in host-I/O steps the device copies of
        obs/reward/flags are not written."""
        N, A = self.num_envs, max(1, self.action_dim)
        if getattr(self, "_h_action", None) is None:
            self._h_action = torch.zeros((N, A), dtype=torch.float32).pin_memory()
            self._h_action_np = self._h_action.numpy()  # a view of the pinned buffer
            outs = self._host_outputs()
            # the arena's tensors come back in one copy; frames (render modes) one copy each
            self._h_arena = torch.zeros(self._out_arena.numel(), dtype=torch.uint8).pin_memory()
            hv = self._arena_views(self._h_arena)
            self._h_in_arena = {k: ("obs" if k in ("obs", "obs/state") else k) for k in outs
                                if k in ("obs", "obs/state", "reward", "terminated", "truncated", "success", "fail")}
            self._h_outs = {k: hv[self._h_in_arena[k]] if k in self._h_in_arena
                            else torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in outs.items()}
            self._h_dev_outs = outs
            # zero-copy: the step kernel reads the actions from, and writes obs / reward / flags to,
            # the pinned host buffers directly over PCIe (page-locked memory is device-addressable
            # under UVA), so the graph has no H2D/D2H copy nodes for them; frames are still copied
            self._c_out_host = cabi.BsStepOutputs.from_buffer_copy(self.c_out)
            for k in ("reward", "terminated", "truncated", "success", "fail"):
                setattr(self._c_out_host, k, hv[k].data_ptr())
            self._c_out_host.obs = hv["obs"].data_ptr()

        # frames that are plain views of the renderer's buffers (env-major) are copied chunk by
        # chunk while the next env chunk renders (a side stream; the D2H copies bound the render
        # configs' e2e, so overlapping the render with them shortens the step); derived entries
        # (pointcloud mask, multi-camera concatenations) are copied after the last chunk
        chunks = self._host_render_chunks()
        views = {}
        if chunks > 1:
            bufs = self.renderer.buffer_storages()
            views = {k: v for k, v in self._flatten_obs(self._obs()).items()
                     if k not in self._h_in_arena and v.untyped_storage().data_ptr() in bufs
                     and v.shape[0] == N}
            if getattr(self, "_copy_stream", None) is None:
                self._copy_stream = torch.cuda.Stream(device=self.device)

        def launch():
            nat.call("bs_step", ctypes.byref(self.scene.c_tables), ctypes.byref(self.scene.c_state),
                     ctypes.byref(self._c_out_host), ctypes.byref(self.c_params), self._h_action.data_ptr(),
                     nat.stream_handle())
            if views:
                main, side = torch.cuda.current_stream(self.device), self._copy_stream

                def after_chunk(a, b):
                    side.wait_stream(main)  # this chunk's frames are rendered
                    with torch.cuda.stream(side):
                        for k, v in views.items():
                            self._h_outs[k][a:b].copy_(v[a:b], non_blocking=True)
                self.renderer.render_chunks(self.scene, chunks, after_chunk)
                main.wait_stream(side)
            else:
                self._render()
            # observation entries derived on the device (the pointcloud validity mask, multi-camera
            # concatenations) are recomputed inside the captured region, not read from the
            # tensors of the capture-time call
            cur = self._flatten_obs(self._obs()) if self.renderer is not None else {}
            for k, v in self._h_dev_outs.items():
                if k not in self._h_in_arena and k not in views:
                    self._h_outs[k].copy_(cur.get(k, v), non_blocking=True)

        self._warm_launchers(lambda: self._launch_step(self.action_buf.data_ptr()))
        self._host_graph = self._capture(launch)
        self._host_graph_key = self._params_key()
        self._host_graph_exec = self._host_graph.raw_cuda_graph_exec()
        self._h_action_ptr = self._h_action.data_ptr()
        self._dev_index = torch.device(self.device).index if torch.device(self.device).index is not None \
            else torch.cuda.current_device()
        self._lib = nat.load()

    def _host_render_chunks(self) -> int:
        """Env chunks of the host-I/O render (1: one launch per camera group, copies after it)."""
        if self.renderer is None:
            return 1
        n = int(os.environ.get("BS_HOST_RENDER_CHUNKS", "8"))  # (A/B knob; 4: C3 e2e +5.7%, 8: +6.4%)
        return max(1, min(n, self.num_envs // 128))

    def _arena_bytes(self) -> int:
        n = 0
        for _, shape, dt in self._arena_layout:
            n = (n + 15) // 16 * 16 + math.prod(shape) * torch.empty(0, dtype=dt).element_size()
        return (n + 15) // 16 * 16

    def _arena_views(self, arena) -> dict:
        out, n = {}, 0
        for name, shape, dt in self._arena_layout:
            n = (n + 15) // 16 * 16
            nb = math.prod(shape) * torch.empty(0, dtype=dt).element_size()
            out[name] = arena[n:n + nb].view(dt).view(shape)
            n += nb
        return out

    @staticmethod
    def _flatten_obs(o) -> dict:
        """{"obs/<path>": tensor} of a (nested) observation dict; a bare tensor is "obs"."""
        if not isinstance(o, dict):
            return {"obs": o}
        out = {}

        def walk(d, prefix=""):
            for k, v in d.items():
                if isinstance(v, dict):
                    walk(v, prefix + k + "/")
                else:
                    out["obs/" + prefix + k] = v
        walk(o)
        return out

    def _host_outputs(self) -> dict:
        out = {"reward": self.reward, "terminated": self.terminated, "truncated": self.truncated,
               "success": self.success, "fail": self.fail}
        out.update(self._flatten_obs(self._obs()))
        return out

    def step_host(self, action):
        """Host-resident step: `action` (N, D) array-like on the host -> dict of pinned host
        tensors (obs..., reward, terminated, truncated, success, fail), valid until the next
        call.  One graph launch and one stream synchronisation per step."""
        if self._host_graph is None:
            self.enable_host_io()
        a = action
        if not (type(a) is np.ndarray and a.dtype == np.float32 and a.flags.c_contiguous):
            a = np.ascontiguousarray(action, dtype=np.float32)
        if a.shape != (self.num_envs, self.action_dim):
            raise DimensionError(f"action must have shape ({self.num_envs}, {self.action_dim}), got {a.shape}")
        if self._host_graph_key != self._params_key():
            self.enable_host_io()
        # one C call: stage the actions into the pinned buffer the graph reads (with the exact
        # inf / NaN test, before anything is launched), replay the host-I/O graph on the current
        # stream and wait for it
        st = self._lib.bs_host_step(a.ctypes.data, self._h_action_ptr, a.size, int(self.validate_actions),
                                    self._host_graph_exec, torch._C._cuda_getCurrentRawStream(self._dev_index))
        if st:
            if st == BS_ERR_INPUT:
                raise InputError("non-finite action")
            raise_for_status(st, "bs_host_step")
        return self._h_outs

    def host_io_bytes(self):
        """(H2D, D2H) bytes per step_host call."""
        frames = sum(v.numel() * v.element_size() for v in self._h_outs.values()
                     if v.untyped_storage().data_ptr() != self._h_arena.untyped_storage().data_ptr())
        return self._h_action.numel() * 4, self._h_arena.numel() + frames

    def _obs(self):
        if self.obs_mode == "state":
            return self.state_obs
        out = {"state": self.state_obs}
        if self.renderer is not None:
            out.update(self.renderer.observation(self.obs_mode))
        return out

    def _result(self) -> StepResult:
        info = {"success": self.success, "fail": self.fail, "unsupported_pairs": self.unsupported,
                "elapsed": self.scene.elapsed, "diverged": self.scene.diverged,
                "contact_count": self.contact_count,
                # rows of envs auto-reset this step: the state obs the episode ended in
                "final_obs": self.final_obs,
                "episode": {"done": self.ep_done, "return": self.ep_return_out, "length": self.ep_length_out,
                            "flags": self.ep_flags_out}}
        return StepResult(self._obs(), self.reward, self.terminated, self.truncated, info)

    def contacts(self):
        """The ContactSet of the last substep: per env a count, shape-slot
        pairs, and point/normal/depth rows."""
        return self.contact_count, self.contact_pairs, self.contact_geom
