"""Task registry and ``make_task``.

Tasks on the hot path (BASELINE.json configs):
  * ``PickCube`` -- PickCube-style tabletop (A-17): ARM3 on a fixed base, one free
    cube on the ground plane, goal on the table; PushCube's success predicate
    (cube within 2.5 cm of the goal in xy), dense reward
    -(|ee - cube| + |cube_xy - goal_xy|), time limit 100.
  * ``OpenCabinet`` -- ARM3 + a synthetic cabinet with per-env 2-6 drawers/doors (A-18,
    OpenChain-Hetero SPEC.md:615): success = target joint qpos > 0.9 * upper limit.
  * ``PickHetero`` -- per-env object kind/size/colour and two jittered cameras (config C5).
  * ``CartpoleBalance`` -- the cartpole fixture: slider driven, hinge passive,
    reward cos(theta), success = upright for the trailing 50 steps, obs (x, x_dot, theta, theta_dot).
"""

from __future__ import annotations

from dataclasses import replace

from . import cabi
from .descriptors import (CartpoleSpec, OpenCabinetSpec, PickCubeSpec, PickHeteroSpec, SceneDesc,  # noqa: F401
                          cartpole_desc, hetero_descs, hetero_objects, opencabinet_descs, pickcube_desc)
from .envs import Env, SimConfig
from .scene import build_batch


def pickcube_scene(spec: PickCubeSpec) -> SceneDesc:
    return pickcube_desc(spec)


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


@register("OpenCabinet")
def _make_opencabinet(num_envs, seed, overrides, obs_mode, device, shard, sim, cameras, **kw):
    spec = replace(OpenCabinetSpec(), **(overrides or {}))
    descs = opencabinet_descs(spec, num_envs, seed)
    scene = build_batch(descs, seed, spec.control(), device, shard)
    ee = scene.models[0].link_names.index(f"arm/{spec.ee_link}")
    renderer = _renderer(scene, obs_mode, cameras, seed)
    env = Env(scene, cabi.TASK_OPENCHAIN, spec.task_f(), ee, spec.max_steps, seed, sim, obs_mode, renderer,
              name="OpenCabinet", **kw)
    env.spec = spec
    env.descs = descs
    env.reset()
    return env


@register("PickHetero")
def _make_pickhetero(num_envs, seed, overrides, obs_mode, device, shard, sim, cameras, **kw):
    import numpy as np

    from .cameras import CameraConfig, CameraJitter, look_at, pinhole

    spec = replace(PickHeteroSpec(), **(overrides or {}))
    descs = hetero_descs(spec, num_envs, seed)
    scene = build_batch(descs, seed, spec.control(), device, shard)
    ee = scene.models[0].link_names.index(f"arm/{spec.ee_link}")
    renderer = None
    if obs_mode != "state":
        res = spec.camera_res
        if cameras is None:
            views = [("base_camera", (0.15, 0.5, 0.4)), ("side_camera", (0.15, -0.5, 0.4))]
            cameras = [CameraConfig(n, pose_p=eye, pose_q=look_at(eye, (-0.15, 0.0, 0.02)), **pinhole(res, res, 60.0))
                       for n, eye in views]
        objs = hetero_objects(spec, num_envs, seed)[scene.env_offset:scene.env_offset + scene.num_envs]
        colors = scene.host_tables["shape_color"][scene.model_index, :, :3].astype(np.float32).copy()
        for e, (_, _, rgb) in enumerate(objs):
            pm = scene.models[scene.model_index[e]]
            for s_idx, sh in enumerate(pm.shapes):
                if sh["btype"] == cabi.BODY_ACTOR:
                    colors[e, s_idx] = rgb
        renderer = _renderer(scene, obs_mode, cameras, seed,
                             CameraJitter(spec.camera_pos_jitter, spec.camera_rot_jitter, 0.0), colors)
    env = Env(scene, cabi.TASK_PICKCUBE, spec.task_f(), ee, spec.max_steps, seed, sim, obs_mode, renderer,
              name="PickHetero", **kw)
    env.spec = spec
    env.descs = descs
    env.reset()
    return env


@register("CartpoleBalance")
def _make_cartpole(num_envs, seed, overrides, obs_mode, device, shard, sim, cameras, **kw):
    from .cameras import CameraConfig, look_at, pinhole

    spec = replace(CartpoleSpec(), **(overrides or {}))
    scene = build_batch([cartpole_desc(spec)] * num_envs, seed, spec.control(), device, shard)
    if obs_mode != "state" and cameras is None:
        eye = (0.0, -3.0, 0.6)
        cameras = [CameraConfig("front_camera", pose_p=eye, pose_q=look_at(eye, (0.0, 0.0, 0.3)),
                                **pinhole(128, 128, 60.0))]
    renderer = _renderer(scene, obs_mode, cameras, seed)
    env = Env(scene, cabi.TASK_CARTPOLE, spec.task_f(), -1, spec.max_steps, seed, sim, obs_mode, renderer,
              name="CartpoleBalance", **kw)
    env.spec = spec
    env.reset()
    return env


def _renderer(scene, obs_mode, cameras, seed, jitter=None, env_color=None):
    if obs_mode == "state":
        return None
    from .cameras import CameraJitter
    from .render import Renderer, default_cameras

    return Renderer(scene, cameras if cameras is not None else default_cameras(), obs_mode, seed,
                    jitter or CameraJitter(), env_color=env_color)


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
    env = TASKS[name](num_envs, seed, overrides, obs_mode, device, shard, sim, cameras, **kw)
    env.task_name = name
    env.overrides = dict(overrides or {})
    env.global_num_envs = num_envs
    env.shard = tuple(shard) if shard is not None else None
    env.custom_cameras = list(cameras) if cameras is not None else None
    return env
