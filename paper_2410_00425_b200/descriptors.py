"""Per-env scene descriptors (SPEC.md:186-194 ``build_batch`` input).

Plain data: which articulation templates sit where, which free actors and static shapes an
env contains.  Envs may differ (heterogeneous batches); the packer
(``scene.py``) groups identical layouts into shared device tables.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .assets import ArticulationTemplate


@dataclass(frozen=True)
class ArticulationDesc:
    name: str
    template: ArticulationTemplate
    base_p: tuple = (0.0, 0.0, 0.0)
    base_q: tuple = (1.0, 0.0, 0.0, 0.0)

    def key(self):
        return ("art", self.name, self.template.to_json(), tuple(self.base_p), tuple(self.base_q))


@dataclass(frozen=True)
class ActorDesc:
    """A free rigid body with one primitive shape; its origin is its centre of mass."""

    name: str
    kind: str
    size: tuple
    density: float = 1000.0
    color: tuple = (0.6, 0.6, 0.6, 1.0)

    def key(self):
        return ("actor", self.name, self.kind, tuple(self.size), self.density, tuple(self.color))


@dataclass(frozen=True)
class StaticDesc:
    """Immovable shape in world coordinates (e.g. the ground plane, local +z = normal)."""

    name: str
    kind: str
    size: tuple = ()
    pos: tuple = (0.0, 0.0, 0.0)
    quat: tuple = (1.0, 0.0, 0.0, 0.0)
    color: tuple = (0.4, 0.4, 0.4, 1.0)

    def key(self):
        return ("static", self.name, self.kind, tuple(self.size), tuple(self.pos), tuple(self.quat),
                tuple(self.color))


def actor_rest_pose(kind: str, size) -> tuple:
    """Resting height and orientation of a free primitive on the ground plane (DESIGN.md
    A-26): boxes and spheres upright at their half-height / radius; capsules and cylinders
    lie on their side (local z axis rotated onto world x)."""
    if kind == "box":
        return (float(size[2]), 1.0, 0.0, 0.0, 0.0)
    if kind == "sphere":
        return (float(size[0]), 1.0, 0.0, 0.0, 0.0)
    if kind in ("capsule", "cylinder"):
        h = math.sqrt(0.5)
        return (float(size[0]), h, 0.0, h, 0.0)
    raise ValueError(f"no resting pose for actor kind {kind!r}")


@dataclass(frozen=True)
class SceneDesc:
    articulations: tuple = ()
    actors: tuple = ()
    statics: tuple = field(default=())

    def key(self):
        return tuple(x.key() for x in (*self.articulations, *self.actors, *self.statics))


GROUND = StaticDesc("ground", "plane", (), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0), (0.45, 0.45, 0.45, 1.0))


@dataclass(frozen=True)
class ControlSpec:
    """Controller preset: which articulation the action drives."""

    mode: str = "pd_joint_delta_pos"
    robot: str = "arm"
    action_scale: float = 0.1
    kp: float = 1000.0
    kd: float = 2.0 * math.sqrt(1000.0)
    force_limit: float = 100.0
    ik_lambda: float = 0.05
    action_scale_rot: float = 0.05   # pd_ee_delta_pose rotation, rad per unit action (A-22)
    joints: tuple = ()               # joint subset by name; empty = every dof of `robot`


@dataclass(frozen=True)
class PickCubeSpec:
    """PickCube-style tabletop (A-17): numbers shared by the product and the oracle."""

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


def pickcube_desc(spec: PickCubeSpec) -> SceneDesc:
    """ARM3 (tasks/fixtures.py:83-152) on a fixed base + one free cube + the ground plane."""
    from . import fixtures as F
    from .assets import load_urdf

    arm = ArticulationDesc("arm", load_urdf(F.ARM3_URDF), tuple(spec.arm_base_p))
    cube = ActorDesc("cube", "box", (spec.cube_half,) * 3, spec.cube_density, spec.cube_color)
    return SceneDesc((arm,), (cube,), (GROUND,))


@dataclass(frozen=True)
class OpenCabinetSpec:
    """Articulated-object task (BASELINE config 4; OpenChain-Hetero; A-18):
    ARM3 on a fixed base facing a synthetic cabinet whose part count (2-6) and kinds
    (prismatic drawer 'd' / revolute door 'r') are sampled per env at build time; one part is
    the per-episode target; success = target joint qpos > 0.9 * upper limit."""

    arm_base_p: tuple = (-0.5, 0.0, 0.25)
    q_rest: tuple = (0.0, -0.3, 1.2)
    q_noise: float = 0.02
    cabinet_p: tuple = (0.1, 0.0, 0.0)
    cabinet_yaw: float = math.pi            # front face (+x of the cabinet) towards the arm
    min_parts: int = 2
    max_parts: int = 6
    success_frac: float = 0.9
    max_steps: int = 100
    ee_link: str = "ee"
    control_mode: str = "pd_joint_delta_pos"
    action_scale: float = 0.1
    kp: float = 1000.0
    kd: float = 2.0 * math.sqrt(1000.0)
    force_limit: float = 100.0

    def task_f(self):
        return [self.q_noise, self.success_frac, 0.0, 0.0, 0.0, 0.0, *self.q_rest]

    def control(self):
        return ControlSpec(self.control_mode, "arm", self.action_scale, self.kp, self.kd, self.force_limit)


@dataclass(frozen=True)
class CartpoleSpec:
    """CartpoleBalance (PAPER.md A.10): the cartpole fixture (tasks/fixtures.py:154-176)
    alone, the slider driven by pd_joint_delta_pos, the hinge passive.  Reset: slider, hinge and
    both rates ~ U[-init_noise, init_noise].  Reward = cos(hinge angle) (upright cosine shaping).
    Success = |angle| < success_angle on each of the trailing `success_steps` control steps (a
    per-env streak counter).  Fail = |angle| > fail_angle or |slider| > fail_x (or divergence).
    State obs = (x, x_dot, theta, theta_dot)."""

    init_noise: float = 0.05
    success_angle: float = 0.2
    success_steps: int = 50
    fail_angle: float = 0.8
    fail_x: float = 1.7
    max_steps: int = 200
    control_mode: str = "pd_joint_delta_pos"
    action_scale: float = 0.01   # m per unit action (target velocity = 0.6 m/s per unit action)
    kp: float = 1000.0
    kd: float = 2.0 * math.sqrt(1000.0)
    force_limit: float = 100.0

    def task_f(self):
        return [self.init_noise, self.success_angle, float(self.success_steps), self.fail_angle, self.fail_x,
                0.0, 0.0, 0.0, 0.0]

    def control(self):
        return ControlSpec(self.control_mode, "cartpole", self.action_scale, self.kp, self.kd, self.force_limit,
                           joints=("slider",))


def cartpole_desc(spec: CartpoleSpec) -> SceneDesc:
    from . import fixtures as F
    from .assets import load_mjcf

    return SceneDesc((ArticulationDesc("cartpole", load_mjcf(F.CARTPOLE_MJCF)[0]),), (), ())


TAG_SCENE = 0x5343454E  # 'SCEN': build-time per-env scene sampling stream


def cabinet_kinds(spec: OpenCabinetSpec, num_envs: int, seed: int, env_offset: int = 0):
    """Per-env part strings, drawn from each env's counter stream (shard-invariant)."""
    from . import rng

    ids = np.arange(env_offset, env_offset + num_envs, dtype=np.uint64)
    u = rng.uniforms(seed, ids, 0, TAG_SCENE, 1 + spec.max_parts)
    span = spec.max_parts - spec.min_parts + 1
    out = []
    for e in range(num_envs):
        n = spec.min_parts + min(int(u[e, 0] * span), span - 1)
        out.append("".join("d" if u[e, 1 + i] < 0.5 else "r" for i in range(n)))
    return out


def opencabinet_descs(spec: OpenCabinetSpec, num_envs: int, seed: int):
    """One SceneDesc per env (heterogeneous): ARM3 + cabinet(kinds) + ground."""
    from . import fixtures as F
    from .assets import load_urdf

    arm = ArticulationDesc("arm", load_urdf(F.ARM3_URDF), tuple(spec.arm_base_p))
    h = 0.5 * spec.cabinet_yaw
    cq = (math.cos(h), 0.0, 0.0, math.sin(h))
    cache = {}
    descs = []
    for kinds in cabinet_kinds(spec, num_envs, seed):
        if kinds not in cache:
            cab = ArticulationDesc("cabinet", load_urdf(F.make_cabinet_urdf(kinds)), tuple(spec.cabinet_p), cq)
            cache[kinds] = SceneDesc((arm, cab), (), (GROUND,))
        descs.append(cache[kinds])
    return descs


@dataclass(frozen=True)
class PickHeteroSpec(PickCubeSpec):
    """Heterogeneous tabletop (BASELINE config 5): every env gets its own object
    kind (sphere / box / capsule -- the SPEC.md:339 pair set), size level in
    [size_lo, size_hi] and colour (texture randomisation), and its own jittered
    cameras (+-2 cm, +-2 deg)."""

    kinds: tuple = ("sphere", "box", "capsule")
    size_lo: float = 0.015
    size_hi: float = 0.035
    size_levels: int = 9
    camera_res: int = 256
    camera_pos_jitter: float = 0.02
    camera_rot_jitter: float = math.radians(2.0)


def hetero_objects(spec: PickHeteroSpec, num_envs: int, seed: int, env_offset: int = 0):
    """Per-env (kind, size tuple, rgb) from each env's build-time counter stream."""
    from . import rng

    ids = np.arange(env_offset, env_offset + num_envs, dtype=np.uint64)
    u = rng.uniforms(seed, ids, 1, TAG_SCENE, 5)
    out = []
    nk, nl = len(spec.kinds), spec.size_levels
    for e in range(num_envs):
        kind = spec.kinds[min(int(u[e, 0] * nk), nk - 1)]
        lev = min(int(u[e, 1] * nl), nl - 1)
        sz = spec.size_lo + lev * (spec.size_hi - spec.size_lo) / max(nl - 1, 1)
        size = {"sphere": (sz,), "box": (sz, sz, sz), "capsule": (sz, sz)}[kind]
        out.append((kind, size, (float(u[e, 2]), float(u[e, 3]), float(u[e, 4]))))
    return out


def hetero_descs(spec: PickHeteroSpec, num_envs: int, seed: int):
    """One SceneDesc per env: ARM3 + that env's object + ground (colours are per-env render
    inputs, not part of the layout, so envs with the same kind/size share a model)."""
    from . import fixtures as F
    from .assets import load_urdf

    arm = ArticulationDesc("arm", load_urdf(F.ARM3_URDF), tuple(spec.arm_base_p))
    cache = {}
    descs = []
    for kind, size, _ in hetero_objects(spec, num_envs, seed):
        key = (kind, size)
        if key not in cache:
            obj = ActorDesc("object", kind, size, spec.cube_density, (0.5, 0.5, 0.5, 1.0))
            cache[key] = SceneDesc((arm,), (obj,), (GROUND,))
        descs.append(cache[key])
    return descs
