"""Oracle scene model: per-env-model tables built straight from templates + descriptors.

Test infrastructure (see oracle/__init__.py).  Built independently of the product's packer
(paper_2410_00425_b200/scene.py) so a packing bug cannot hide behind a shared table.

One Model = one distinct env layout (forest of fixed-base articulations, free actors,
static shapes).  Link order: articulations in descriptor order, each in template order
(topological).  Shape slot order (decision A-5): link shapes (link order, then
per-link order), actor shapes, static shapes last -- so the static body is always the
second body of a pair and the normal points into the dynamic one (A-25).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import se3

KIND = {"sphere": 0, "box": 1, "capsule": 2, "cylinder": 3, "plane": 4}
SPHERE, BOX, CAPSULE, CYLINDER, PLANE = range(5)
FIXED, REVOLUTE, PRISMATIC = 0, 1, 2
BODY_LINK, BODY_ACTOR, BODY_STATIC = 0, 1, 2

# Supported narrowphase pairs keyed by sorted (kind_a, kind_b) -> max contacts.
PAIR_MAX = {
    (SPHERE, PLANE): 1,
    (BOX, PLANE): 4,
    (SPHERE, SPHERE): 1,
    (SPHERE, BOX): 1,
    (CAPSULE, PLANE): 2,
}


def bounding_radius(kind: int, size) -> float:
    if kind == SPHERE:
        return size[0]
    if kind == BOX:
        return math.sqrt(size[0] ** 2 + size[1] ** 2 + size[2] ** 2)
    if kind == CAPSULE:
        return size[0] + size[1]
    if kind == CYLINDER:
        return math.sqrt(size[0] ** 2 + size[1] ** 2)
    return math.inf


@dataclass
class Pair:
    i: int          # first shape slot (body A)
    j: int          # second shape slot (body B)
    kind: tuple     # (kind_first_role, kind_second_role) of the supported routine, or None
    swap: bool      # routine computed with roles (j, i); normal is flipped back
    maxc: int       # candidate contact slots (0 = unsupported pair, counted)


class Model:
    """Numpy tables for one env layout."""

    def __init__(self, desc):
        arts = list(desc.articulations)
        parent, jtype, art, axis, org_p, org_q = [], [], [], [], [], []
        mass, com, inertia, lower, upper, damping, dof_link, dof_of = [], [], [], [], [], [], [], []
        names = []
        shapes = []
        for a_idx, ad in enumerate(arts):
            tpl = ad.template
            base = len(parent)
            pj = {j.child_link: j for j in tpl.joints}
            for k, lk in enumerate(tpl.links):
                names.append(f"{ad.name}/{lk.name}")
                art.append(a_idx)
                if k == tpl.root_link_index:
                    parent.append(-1)
                    jtype.append(FIXED)
                    axis.append((0.0, 0.0, 1.0))
                    org_p.append(tuple(ad.base_p))
                    org_q.append(tuple(ad.base_q))
                    dof_of.append(-1)
                else:
                    j = pj[k]
                    parent.append(base + j.parent_link)
                    jtype.append({"fixed": FIXED, "revolute": REVOLUTE, "prismatic": PRISMATIC}[j.joint_type])
                    axis.append(tuple(j.axis))
                    org_p.append(tuple(j.origin.pos))
                    org_q.append(tuple(j.origin.quat))
                    if j.is_movable:
                        dof_of.append(len(dof_link))
                        dof_link.append(base + k)
                        lower.append(j.limits[0])
                        upper.append(j.limits[1])
                        damping.append(j.damping)
                    else:
                        dof_of.append(-1)
                mass.append(lk.mass)
                com.append(tuple(lk.inertial_origin.pos))
                r = se3.qmat(se3.qnorm(np.asarray(lk.inertial_origin.quat, np.float64)))
                inertia.append(r @ lk.inertia_matrix() @ r.T)
                for s in lk.collision_shapes:
                    shapes.append((BODY_LINK, base + k, s))
        self.L = len(parent)
        self.parent = np.asarray(parent, np.int64)
        self.jtype = np.asarray(jtype, np.int64)
        self.art = np.asarray(art, np.int64)
        self.axis = np.asarray(axis, np.float64).reshape(-1, 3)
        self.org_p = np.asarray(org_p, np.float64).reshape(-1, 3)
        self.org_q = se3.qnorm(np.asarray(org_q, np.float64).reshape(-1, 4)) if self.L else np.zeros((0, 4))
        self.mass = np.asarray(mass, np.float64)
        self.com = np.asarray(com, np.float64).reshape(-1, 3)
        self.inertia = np.asarray(inertia, np.float64).reshape(-1, 3, 3)
        self.dof_of = np.asarray(dof_of, np.int64)
        self.dof_link = np.asarray(dof_link, np.int64)
        self.D = len(dof_link)
        self.lower = np.asarray(lower, np.float64)
        self.upper = np.asarray(upper, np.float64)
        self.damping = np.asarray(damping, np.float64)
        self.link_names = names
        # link is "grounded" when no movable joint lies between it and the world
        grounded = []
        for l in range(self.L):
            p = self.parent[l]
            grounded.append(self.jtype[l] == FIXED and (p < 0 or grounded[p]))
        self.grounded = np.asarray(grounded, bool)
        # actors: one primitive shape each, origin at the COM
        self.A = len(desc.actors)
        self.actor_mass = np.zeros(self.A)
        self.actor_inertia = np.zeros((self.A, 3))
        for a_idx, ac in enumerate(desc.actors):
            m, diag = primitive_mass(ac.kind, ac.size, ac.density)
            self.actor_mass[a_idx] = m
            self.actor_inertia[a_idx] = diag
            shapes.append((BODY_ACTOR, a_idx, ac))
        for s_idx, st in enumerate(desc.statics):
            shapes.append((BODY_STATIC, s_idx, st))
        self._pack_shapes(shapes, desc)
        self._pairs()

    def _pack_shapes(self, shapes, desc):
        S = len(shapes)
        self.S = S
        self.s_btype = np.zeros(S, np.int64)
        self.s_body = np.zeros(S, np.int64)
        self.s_kind = np.zeros(S, np.int64)
        self.s_size = np.zeros((S, 3))
        self.s_fp = np.zeros((S, 3))
        self.s_fq = np.tile([1.0, 0.0, 0.0, 0.0], (S, 1))
        self.s_seg = np.zeros(S, np.int64)
        self.s_color = np.zeros((S, 4))
        self.s_radius = np.zeros(S)
        n_links = self.L
        for k, (bt, bi, s) in enumerate(shapes):
            self.s_btype[k] = bt
            self.s_body[k] = bi
            if bt == BODY_LINK:
                kind, size, fp, fq = KIND[s.kind], s.size, s.frame.pos, s.frame.quat
                seg = 1 + bi
                color = desc_link_color(desc, self, bi)
            elif bt == BODY_ACTOR:
                kind, size, fp, fq = KIND[s.kind], s.size, (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0)
                seg = 1 + n_links + bi
                color = s.color
            else:
                kind, size, fp, fq = KIND[s.kind], s.size, s.pos, s.quat
                seg = 1 + n_links + self.A + bi
                color = s.color
            self.s_kind[k] = kind
            self.s_size[k, :len(size)] = size
            self.s_fp[k] = fp
            self.s_fq[k] = se3.qnorm(np.asarray(fq, np.float64))
            self.s_seg[k] = seg
            self.s_color[k] = color
            self.s_radius[k] = bounding_radius(kind, self.s_size[k])

    def immovable(self, slot: int) -> bool:
        bt = self.s_btype[slot]
        return bt == BODY_STATIC or (bt == BODY_LINK and self.grounded[self.s_body[slot]])

    def _pairs(self):
        pairs = []
        for i in range(self.S):
            for j in range(i + 1, self.S):
                if self.immovable(i) and self.immovable(j):
                    continue
                bi, bj = self.s_btype[i], self.s_btype[j]
                if bi == BODY_LINK and bj == BODY_LINK and \
                        self.art[self.s_body[i]] == self.art[self.s_body[j]]:
                    continue  # same articulation: ignored
                ki, kj = int(self.s_kind[i]), int(self.s_kind[j])
                if (ki, kj) in PAIR_MAX:
                    pairs.append(Pair(i, j, (ki, kj), False, PAIR_MAX[(ki, kj)]))
                elif (kj, ki) in PAIR_MAX:
                    pairs.append(Pair(i, j, (kj, ki), True, PAIR_MAX[(kj, ki)]))
                else:
                    pairs.append(Pair(i, j, None, False, 0))
        self.pairs = pairs
        self.C = sum(p.maxc for p in pairs)


def desc_link_color(desc, model, link_index):
    k = 0
    for ad in desc.articulations:
        n = len(ad.template.links)
        if link_index < k + n:
            return tuple(ad.template.links[link_index - k].visual_color)
        k += n
    raise IndexError(link_index)


def primitive_mass(kind: str, size, density: float):
    """Mass and body-frame principal inertia of a solid primitive (axis along local z)."""
    if kind == "sphere":
        r = size[0]
        m = density * 4.0 / 3.0 * math.pi * r ** 3
        return m, np.full(3, 0.4 * m * r * r)
    if kind == "box":
        hx, hy, hz = size
        m = density * 8.0 * hx * hy * hz
        return m, m / 3.0 * np.array([hy * hy + hz * hz, hx * hx + hz * hz, hx * hx + hy * hy])
    if kind in ("capsule", "cylinder"):
        r, hl = size[0], size[1]
        mc = density * math.pi * r * r * 2.0 * hl
        if kind == "cylinder":
            side = mc * (3.0 * r * r + 4.0 * hl * hl) / 12.0
            return mc, np.array([side, side, 0.5 * mc * r * r])
        ms = density * 4.0 / 3.0 * math.pi * r ** 3
        # cylinder + two hemispheres (hemisphere COM offset 3r/8 from the cap plane)
        iz = 0.5 * mc * r * r + 0.4 * ms * r * r
        ix = mc * (3.0 * r * r + 4.0 * hl * hl) / 12.0 + ms * (0.4 * r * r + hl * hl + 0.75 * hl * r)
        return mc + ms, np.array([ix, ix, iz])
    raise ValueError(f"actor kind {kind!r} has no mass model")
