"""Per-env scene descriptors (SPEC.md:186-194 ``build_batch`` input).

Plain data: which articulation templates sit where, which free actors and static shapes an
env contains.  Envs may differ (heterogeneous batches); the packer
(``scene.py``) groups identical layouts into shared device tables.
"""

from __future__ import annotations

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
