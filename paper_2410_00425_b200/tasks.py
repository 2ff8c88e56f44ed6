"""Task registry and ``make_task``.

Tasks on the hot path (BASELINE.json configs):
  * ``PickCube`` -- PickCube-style tabletop (A-17): ARM3 on a fixed base, one free
    cube on the ground plane, goal on the table; PushCube's success predicate
    (cube within 2.5 cm of the goal in xy), dense reward
    -(|ee - cube| + |cube_xy - goal_xy|), time limit 100.
  * ``OpenCabinet`` -- ARM3 + a synthetic cabinet with per-env 2-6 drawers/doors (A-18,
    OpenChain-Hetero SPEC.md:615): success = target joint qpos > 0.9 * upper limit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

from . import cabi
from . import fixtures as F
from .assets import load_urdf
from .descriptors import GROUND, ActorDesc, ArticulationDesc, SceneDesc
from .envs import Env, SimConfig
from .scene import ControlSpec, build_batch


@dataclass(frozen=True)
class PickCubeSpec:
    arm_base_p: tuple = (-0.5, 0.0, 0.25)
    q_rest: tuple = (0.0, -0.3, 1.2)
    q_noise: float = 0.02
    cube_half: float = 0.02
    cube_density: float = 1000.0
    cube_color: tuple = (0.2, 0.4, 0.9, 1.0)
    cube_xy: float = 0.1
    goal_xy: float = 0.1
    success_dist: float = 0.025
    fail_z: float = -0.1
    max_steps: int = 100
    ee_link: str = "ee"
    control_mode: str = "pd_joint_delta_pos"
    action_scale: float = 0.1
    kp: float = 1000.0
    kd: float = 2.0 * math.sqrt(1000.0)
    force_limit: float = 100.0

    def task_f(self):
        return [self.q_noise, self.cube_half, self.cube_xy, self.goal_xy, self.success_dist, self.fail_z,
                *self.q_rest]

    def control(self):
        return ControlSpec(self.control_mode, "arm", self.action_scale, self.kp, self.kd, self.force_limit)


def pickcube_scene(spec: PickCubeSpec) -> SceneDesc:
    arm = ArticulationDesc("arm", load_urdf(F.ARM3_URDF), tuple(spec.arm_base_p))
    cube = ActorDesc("cube", "box", (spec.cube_half,) * 3, spec.cube_density, spec.cube_color)
    return SceneDesc((arm,), (cube,), (GROUND,))


TASKS = {}


def register(name):
    def deco(fn):
        TASKS[name] = fn
        return fn
    return deco


@register("PickCube")
def _make_pickcube(num_envs, seed, overrides, obs_mode, device, shard, sim, cameras, **kw):
    spec = replace(PickCubeSpec(), **(overrides or {}))
    desc = pickcube_scene(spec)
    scene = build_batch([desc] * num_envs, seed, spec.control(), device, shard)
    ee = scene.models[0].link_names.index(f"arm/{spec.ee_link}")
    renderer = _renderer(scene, obs_mode, cameras, seed)
    env = Env(scene, cabi.TASK_PICKCUBE, spec.task_f(), ee, spec.max_steps, seed, sim, obs_mode, renderer,
              name="PickCube", **kw)
    env.spec = spec
    env.reset()
    return env


def _renderer(scene, obs_mode, cameras, seed):
    if obs_mode == "state":
        return None
    from .render import Renderer, default_cameras

    return Renderer(scene, cameras if cameras is not None else default_cameras(), obs_mode, seed)


def make_task(name: str, num_envs: int, seed: int = 0, overrides=None, obs_mode: str = "state", device=None,
              shard=None, sim: SimConfig = None, cameras=None, **kw) -> Env:
    """Build a registered task with `num_envs` parallel envs on the current GPU.

    `shard=(rank, world)`: this process owns global envs [rank*N/world, (rank+1)*N/world)
    of an N-env batch (layout maxima and RNG keys are global, so shards compose bitwise).
    """
    if name not in TASKS:
        raise KeyError(f"unknown task {name!r}; registered: {sorted(TASKS)}")
    if num_envs < 1:
        raise ValueError("num_envs must be >= 1")
    return TASKS[name](num_envs, seed, overrides, obs_mode, device, shard, sim, cameras, **kw)
