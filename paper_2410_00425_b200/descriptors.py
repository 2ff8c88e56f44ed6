"""Per-env scene descriptors (SPEC.md:186-194 ``build_batch`` input).

Plain data: which articulation templates sit where, which free actors and static shapes an
env contains.  Envs may differ (heterogeneous batches); the packer
(``scene.py``) groups identical layouts into shared device tables.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

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
