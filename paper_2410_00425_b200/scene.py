"""SoA GPU scene store: the B200 replacement for the reference's SceneBatch.

``build_batch`` packs per-env descriptors into

* model tables -- one copy per DISTINCT env layout (links in topological order, dof
  parameters, shapes, the static pair list with narrowphase routine codes, actors),
  padded to global maxima ``L_max/D_max/S_max/P_max/A_max/C_max`` so every env row has
  the same stride (padding + masks, not ragged storage);
* state rows -- qpos/qvel (N, D_max), actor pose/velocity (N, A_max, 7|6), the link-pose
  cache (N, L_max, 7), task goal, episode counters; masked-out entries stay zero;

all as CUDA tensors owned by Python (the kernels never allocate).  The same structs are
handed to every C-ABI call, so a step is a single launch with no host work.

Views are resolved once by name into per-env index tensors; their
accessors are gathers on the device (no string lookup in the step path).
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import cabi
from . import hostmath as hm
from .descriptors import ControlSpec, SceneDesc, actor_rest_pose  # noqa: F401
from .errors import DimensionError, LayoutMismatchError, SceneBuildError, ViewLookupError


def _bounding_radius(kind, size):
    if kind == "sphere":
        return size[0]
    if kind == "box":
        return math.sqrt(size[0] ** 2 + size[1] ** 2 + size[2] ** 2)
    if kind == "capsule":
        return size[0] + size[1]
    if kind == "cylinder":
        return math.sqrt(size[0] ** 2 + size[1] ** 2)
    return math.inf


def actor_mass_properties(kind, size, density):
    """Solid primitive mass and principal inertia (axis along local z)."""
    if kind == "sphere":
        r = size[0]
        m = density * (4.0 / 3.0) * math.pi * r ** 3
        return m, (0.4 * m * r * r,) * 3
    if kind == "box":
        hx, hy, hz = size
        m = density * 8.0 * hx * hy * hz
        return m, (m / 3.0 * (hy * hy + hz * hz), m / 3.0 * (hx * hx + hz * hz), m / 3.0 * (hx * hx + hy * hy))
    if kind in ("capsule", "cylinder"):
        r, hl = size[0], size[1]
        mc = density * math.pi * r * r * 2.0 * hl
        if kind == "cylinder":
            ix = mc * (3.0 * r * r + 4.0 * hl * hl) / 12.0
            return mc, (ix, ix, 0.5 * mc * r * r)
        ms = density * (4.0 / 3.0) * math.pi * r ** 3
        ix = mc * (3.0 * r * r + 4.0 * hl * hl) / 12.0 + ms * (0.4 * r * r + hl * hl + 0.75 * hl * r)
        return mc + ms, (ix, ix, 0.5 * mc * r * r + 0.4 * ms * r * r)
    raise SceneBuildError(f"actor kind {kind!r} has no mass model")


class PackedModel:
    """Host-side tables of one env layout (numpy), plus its name registry."""

    def __init__(self, desc: SceneDesc, control: ControlSpec):
        self.desc = desc
        links, shapes = [], []
        self.dofs = []          # (link, joint spec, articulation name)
        self.link_names, self.joint_names = [], []
        for art_idx, ad in enumerate(desc.articulations):
            t = ad.template
            base = len(links)
            by_child = {j.child_link: j for j in t.joints}
            for k, lk in enumerate(t.links):
                j = by_child.get(k)
                rec = {"art": art_idx, "parent": -1 if j is None else base + j.parent_link, "link": lk}
                if j is None:
                    rec.update(jtype="fixed", axis=(0.0, 0.0, 1.0), org_p=tuple(ad.base_p),
                               org_q=tuple(hm.qnormalize(ad.base_q)))
                else:
                    rec.update(jtype=j.joint_type, axis=tuple(j.axis), org_p=tuple(j.origin.pos),
                               org_q=tuple(hm.qnormalize(j.origin.quat)))
                    self.joint_names.append((f"{ad.name}/{j.name}", len(links)))
                rec["dof"] = -1
                if j is not None and j.is_movable:
                    rec["dof"] = len(self.dofs)
                    self.dofs.append((len(links), j, ad.name))
                links.append(rec)
                self.link_names.append(f"{ad.name}/{lk.name}")
                for s in lk.collision_shapes:
                    shapes.append({"btype": cabi.BODY_LINK, "body": len(links) - 1, "kind": s.kind,
                                   "size": s.size, "p": s.frame.pos, "q": hm.qnormalize(s.frame.quat),
                                   "color": lk.visual_color})
        self.links = links
        self.L, self.D = len(links), len(self.dofs)
        grounded = []
        for rec in links:
            p = rec["parent"]
            grounded.append(rec["jtype"] == "fixed" and (p < 0 or grounded[p]))
        self.grounded = grounded
        self.actor_names = [a.name for a in desc.actors]
        self.actors = []
        for a_idx, ac in enumerate(desc.actors):
            m, inertia = actor_mass_properties(ac.kind, ac.size, ac.density)
            self.actors.append((m, inertia))
            shapes.append({"btype": cabi.BODY_ACTOR, "body": a_idx, "kind": ac.kind, "size": ac.size,
                           "p": (0.0, 0.0, 0.0), "q": (1.0, 0.0, 0.0, 0.0), "color": ac.color})
        self.static_names = [s.name for s in desc.statics]
        for s_idx, st in enumerate(desc.statics):
            shapes.append({"btype": cabi.BODY_STATIC, "body": s_idx, "kind": st.kind, "size": st.size,
                           "p": st.pos, "q": hm.qnormalize(st.quat), "color": st.color})
        self.A, self.S = len(desc.actors), len(shapes)
        for sh in shapes:
            b = sh["body"]
            sh["seg"] = 1 + (b if sh["btype"] == cabi.BODY_LINK else
                             self.L + b if sh["btype"] == cabi.BODY_ACTOR else self.L + self.A + b)
        self.shapes = shapes
        # entity registry for segmentation ids: links, actors, statics
        self.entities = self.link_names + [f"actor/{n}" for n in self.actor_names] + \
            [f"static/{n}" for n in self.static_names]
        self._pairs()
        self._controls(control)

    def _immovable(self, sh):
        return sh["btype"] == cabi.BODY_STATIC or (sh["btype"] == cabi.BODY_LINK and self.grounded[sh["body"]])

    def _pairs(self):
        pairs = []
        C = 0
        for i, a in enumerate(self.shapes):
            for j in range(i + 1, self.S):
                b = self.shapes[j]
                if self._immovable(a) and self._immovable(b):
                    continue
                if a["btype"] == b["btype"] == cabi.BODY_LINK and \
                        self.links[a["body"]]["art"] == self.links[b["body"]]["art"]:
                    continue
                ka, kb = cabi.KIND[a["kind"]], cabi.KIND[b["kind"]]
                code = cabi.PAIR_CODE.get((ka, kb))
                if code is None and (kb, ka) in cabi.PAIR_CODE:
                    code = cabi.PAIR_CODE[(kb, ka)] | cabi.PAIR_SWAP
                code = code or 0
                C += cabi.PAIR_MAXC.get(code & 15, 0)
                pairs.append((i, j, code))
        self.pairs = pairs
        self.P, self.C = len(pairs), C

    def _controls(self, control: ControlSpec):
        self.ctrl = [-1] * self.D
        self.kp = [0.0] * self.D
        self.kd = [0.0] * self.D
        self.flim = [math.inf] * self.D
        n = 0
        for d, (_, j, art_name) in enumerate(self.dofs):
            if art_name == control.robot and (not control.joints or j.name in control.joints):
                self.ctrl[d] = n
                self.kp[d], self.kd[d], self.flim[d] = control.kp, control.kd, control.force_limit
                if control.mode == "base_forward_rotate":
                    self.kp[d] = 0.0  # the base joints are velocity servos
                n += 1
        self.action_dim = (6 if control.mode == "pd_ee_delta_pose" and n else
                           2 if control.mode == "base_forward_rotate" and n else n)


def _stack(models, fn, width, dtype, fill=0):
    out = np.full((len(models), width) + fn.shape_tail, fill, dtype=dtype) if hasattr(fn, "shape_tail") else None
    return out


class SceneBatch:
    """Padded SoA state of N envs on one device (one shard of the global batch)."""

    def __init__(self, descs, control: ControlSpec = ControlSpec(), device=None, env_offset: int = 0,
                 num_global_envs: int = None, global_descs=None):
        nat.ensure_device(device)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        descs = list(descs)
        if not descs:
            raise SceneBuildError("build_batch needs at least one env descriptor")
        global_descs = list(global_descs) if global_descs is not None else descs
        self.num_envs = len(descs)
        self.env_offset = int(env_offset)
        self.control = control
        # distinct layouts -> models (global, so every shard has the same strides)
        keys, gmodels, gmodel_of = {}, [], []
        for e, d in enumerate(global_descs):
            if not isinstance(d, SceneDesc):
                raise SceneBuildError(f"env {e}: descriptor is not a SceneDesc")
            k = d.key()
            if k not in keys:
                try:
                    keys[k] = len(gmodels)
                    gmodels.append(PackedModel(d, control))
                except Exception as exc:  # noqa: BLE001
                    raise SceneBuildError(f"env {e}: {exc}") from exc
            gmodel_of.append(keys[k])
        self.models = gmodels
        self.L_max = max(1, max(m.L for m in gmodels))
        self.D_max = max(1, max(m.D for m in gmodels))
        self.S_max = max(1, max(m.S for m in gmodels))
        self.P_max = max(1, max(m.P for m in gmodels))
        self.A_max = max(1, max(m.A for m in gmodels))
        self.C_max = max(1, max(m.C for m in gmodels))
        self.action_dim = max(m.action_dim for m in gmodels)
        local = gmodel_of[self.env_offset:self.env_offset + self.num_envs] if global_descs is not descs else gmodel_of
        self.model_index = np.asarray(local, np.int32)
        self.layout_hash = hashlib.sha256(json.dumps(
            [[repr(k) for k in keys], gmodel_of, self.L_max, self.D_max, self.A_max, self.S_max,
             control.__dict__ if hasattr(control, "__dict__") else repr(control)],
            sort_keys=True, default=str).encode()).hexdigest()[:16]
        self._build_tables()
        self._build_state()
        self._views = {}

    # ------------------------------------------------------------------ tables
    def _build_tables(self):
        M, Lm, Dm, Sm, Pm, Am = len(self.models), self.L_max, self.D_max, self.S_max, self.P_max, self.A_max
        i32, f64 = np.int32, np.float64
        t = {k: np.zeros(s, dt) for k, s, dt in [
            ("n_links", (M,), i32), ("n_dof", (M,), i32), ("n_shapes", (M,), i32), ("n_pairs", (M,), i32),
            ("n_actors", (M,), i32), ("link_parent", (M, Lm), i32), ("link_jtype", (M, Lm), i32),
            ("link_dof", (M, Lm), i32), ("link_grounded", (M, Lm), i32), ("link_axis", (M, Lm, 3), f64),
            ("link_org", (M, Lm, 7), f64), ("link_mass", (M, Lm), f64), ("link_com", (M, Lm, 3), f64),
            ("link_inertia", (M, Lm, 6), f64), ("dof_lower", (M, Dm), f64), ("dof_upper", (M, Dm), f64),
            ("dof_damping", (M, Dm), f64), ("dof_kp", (M, Dm), f64), ("dof_kd", (M, Dm), f64),
            ("dof_flim", (M, Dm), f64), ("dof_ctrl", (M, Dm), i32), ("shape_btype", (M, Sm), i32),
            ("shape_body", (M, Sm), i32), ("shape_kind", (M, Sm), i32), ("shape_seg", (M, Sm), i32),
            ("shape_size", (M, Sm, 3), f64), ("shape_frame", (M, Sm, 7), f64), ("shape_radius", (M, Sm), f64),
            ("shape_color", (M, Sm, 4), np.float32), ("pair_i", (M, Pm), i32), ("pair_j", (M, Pm), i32),
            ("pair_code", (M, Pm), i32), ("pair_slot", (M, Pm), i32), ("actor_mass", (M, Am), f64), ("actor_inertia", (M, Am, 3), f64),
            ("actor_rest", (M, Am, 5), f64)]}
        t["link_parent"][:] = -2
        t["link_dof"][:] = -1
        t["dof_ctrl"][:] = -1
        t["link_org"][..., 3] = 1.0
        t["shape_frame"][..., 3] = 1.0
        t["actor_rest"][..., 1] = 1.0
        for m, pm in enumerate(self.models):
            t["n_links"][m], t["n_dof"][m], t["n_shapes"][m] = pm.L, pm.D, pm.S
            t["n_pairs"][m], t["n_actors"][m] = pm.P, pm.A
            for l, rec in enumerate(pm.links):
                t["link_parent"][m, l] = rec["parent"]
                t["link_jtype"][m, l] = cabi.JOINT[rec["jtype"]]
                t["link_dof"][m, l] = rec["dof"]
                t["link_grounded"][m, l] = int(pm.grounded[l])
                t["link_axis"][m, l] = rec["axis"]
                t["link_org"][m, l] = (*rec["org_p"], *rec["org_q"])
                lk = rec["link"]
                t["link_mass"][m, l] = lk.mass
                t["link_com"][m, l] = lk.inertial_origin.pos
                r = hm.qmatrix(hm.qnormalize(lk.inertial_origin.quat))
                I = r @ lk.inertia_matrix() @ r.T
                t["link_inertia"][m, l] = (I[0, 0], I[1, 1], I[2, 2], I[0, 1], I[0, 2], I[1, 2])
            for d, (_, j, _) in enumerate(pm.dofs):
                t["dof_lower"][m, d], t["dof_upper"][m, d] = j.limits
                t["dof_damping"][m, d] = j.damping
                t["dof_kp"][m, d], t["dof_kd"][m, d] = pm.kp[d], pm.kd[d]
                t["dof_flim"][m, d], t["dof_ctrl"][m, d] = pm.flim[d], pm.ctrl[d]
            for s, sh in enumerate(pm.shapes):
                t["shape_btype"][m, s], t["shape_body"][m, s] = sh["btype"], sh["body"]
                t["shape_kind"][m, s], t["shape_seg"][m, s] = cabi.KIND[sh["kind"]], sh["seg"]
                t["shape_size"][m, s, :len(sh["size"])] = sh["size"]
                t["shape_frame"][m, s] = (*sh["p"], *sh["q"])
                t["shape_radius"][m, s] = _bounding_radius(sh["kind"], sh["size"])
                t["shape_color"][m, s] = sh["color"]
            slot = 0
            for p, (i, j, code) in enumerate(pm.pairs):
                t["pair_i"][m, p], t["pair_j"][m, p], t["pair_code"][m, p] = i, j, code
                t["pair_slot"][m, p] = slot
                slot += cabi.PAIR_MAXC.get(code & 15, 0)
            for a, (mass, inertia) in enumerate(pm.actors):
                t["actor_mass"][m, a] = mass
                t["actor_inertia"][m, a] = inertia
                ad = pm.desc.actors[a]
                t["actor_rest"][m, a] = actor_rest_pose(ad.kind, ad.size)
        self.host_tables = t
        # every table lives in ONE device arena (16-byte aligned slices): a model's tables share a
        # few cache lines instead of one caching-allocator block each, so a launch after an L2
        # flush takes fewer first-touch misses (an explicit L2 bulk prefetch of the arena at
        # kernel entry was measured slower: profiles/r02_summary.md)
        offs, o = {}, 0
        for k, v in t.items():
            offs[k] = o
            o += (v.nbytes + 15) & ~15
        host = np.zeros(max(o, 16), np.uint8)
        for k, v in t.items():
            host[offs[k]:offs[k] + v.nbytes] = np.ascontiguousarray(v).view(np.uint8).reshape(-1)
        self.table_arena = torch.as_tensor(host, device=self.device)
        tdt = {np.dtype(np.int32): torch.int32, np.dtype(np.float32): torch.float32,
               np.dtype(np.float64): torch.float64}
        self.tables = {k: self.table_arena[offs[k]:offs[k] + v.nbytes].view(tdt[v.dtype]).view(v.shape)
                       for k, v in t.items()}
        ct = cabi.BsModelTables()
        ct.num_models, ct.L_max, ct.D_max, ct.S_max = M, Lm, Dm, Sm
        ct.P_max, ct.A_max, ct.C_max = Pm, Am, self.C_max
        ct.A_dyn = max(m.A for m in self.models)  # 0 when no model has a free actor (A_max is padded to 1)
        for k, v in self.tables.items():
            setattr(ct, k, v.data_ptr())
        self.c_tables = ct

    # ------------------------------------------------------------------ state
    def _build_state(self):
        N, dev = self.num_envs, self.device
        f64 = dict(dtype=torch.float64, device=dev)
        self.model_id = torch.as_tensor(self.model_index, device=dev).to(torch.int32).contiguous()
        self.qpos = torch.zeros((N, self.D_max), **f64)
        self.qvel = torch.zeros((N, self.D_max), **f64)
        self.target = torch.zeros((N, self.D_max), **f64)
        self.actor_pose = torch.zeros((N, self.A_max, 7), **f64)
        self.actor_pose[..., 3] = 1.0
        self.actor_vel = torch.zeros((N, self.A_max, 6), **f64)
        self.link_pose = torch.zeros((N, self.L_max, 7), **f64)
        self.link_pose[..., 3] = 1.0
        self.goal = torch.zeros((N, 3), **f64)
        self.diverged = torch.zeros(N, dtype=torch.uint8, device=dev)
        self.elapsed = torch.zeros(N, dtype=torch.int32, device=dev)
        self.reset_count = torch.zeros(N, dtype=torch.int32, device=dev)  # read as uint32 on device
        self.target_dof = torch.full((N,), -1, dtype=torch.int32, device=dev)
        self.ep_return = torch.zeros(N, dtype=torch.float64, device=dev)
        self.ep_flags = torch.zeros(N, dtype=torch.uint8, device=dev)
        # dof / actor validity masks
        ndof = torch.as_tensor([self.models[m].D for m in self.model_index], device=dev)
        nact = torch.as_tensor([self.models[m].A for m in self.model_index], device=dev)
        self.dof_mask = torch.arange(self.D_max, device=dev)[None, :] < ndof[:, None]
        self.actor_mask = torch.arange(self.A_max, device=dev)[None, :] < nact[:, None]
        cs = cabi.BsEnvState()
        cs.num_envs, cs.env_offset = N, self.env_offset
        for k in ("model_id", "qpos", "qvel", "target", "actor_pose", "actor_vel", "link_pose", "goal",
                  "diverged", "elapsed", "reset_count", "target_dof", "ep_return", "ep_flags"):
            setattr(cs, k, getattr(self, k).data_ptr())
        self.c_state = cs

    def c_state_slice(self, a: int, b: int):
        """The C state struct of envs [a, b) (pointers into the same rows; env_offset shifted so
        global env indices -- RNG keys -- stay the same)."""
        cs = cabi.BsEnvState()
        cs.num_envs, cs.env_offset = b - a, self.env_offset + a
        for k in ("model_id", "qpos", "qvel", "target", "actor_pose", "actor_vel", "link_pose", "goal",
                  "diverged", "elapsed", "reset_count", "target_dof", "ep_return", "ep_flags"):
            setattr(cs, k, getattr(self, k)[a:].data_ptr())
        return cs

    STATE_FIELDS = ("qpos", "qvel", "target", "actor_pose", "actor_vel", "link_pose", "goal", "diverged",
                    "elapsed", "reset_count", "target_dof", "ep_return", "ep_flags")

    def forward_kinematics(self):
        nat.call("bs_forward_kinematics", ctypes.byref(self.c_tables), ctypes.byref(self.c_state),
                 nat.stream_handle())
        return self.link_pose

    # ------------------------------------------------------------------ snapshots
    def get_state(self) -> dict:
        """StateSnapshot: device copies of every state row + the layout hash."""
        snap = {k: getattr(self, k).clone() for k in self.STATE_FIELDS}
        snap["layout_hash"] = self.layout_hash
        return snap

    def set_state(self, snap: dict, env_mask=None) -> None:
        """Overwrite the selected envs' rows (all when env_mask is None) bit-exactly;
        unselected envs are untouched."""
        if snap.get("layout_hash") != self.layout_hash:
            raise LayoutMismatchError(
                f"snapshot layout {snap.get('layout_hash')} != scene layout {self.layout_hash}")
        mask = None
        if env_mask is not None:
            mask = torch.as_tensor(env_mask, device=self.device).to(torch.uint8).contiguous()
            if mask.shape != (self.num_envs,):
                raise DimensionError(f"env_mask must have shape ({self.num_envs},), got {tuple(mask.shape)}")
        for k in self.STATE_FIELDS:
            dst = getattr(self, k)
            src = snap[k].to(self.device)
            if src.shape != dst.shape or src.dtype != dst.dtype:
                raise LayoutMismatchError(f"snapshot field {k} has shape {tuple(src.shape)}, expected {tuple(dst.shape)}")
            src = src.contiguous()
            row = dst[0].numel() * dst.element_size() if dst.ndim > 1 else dst.element_size()
            nat.call("bs_masked_copy", src.data_ptr(), dst.data_ptr(), self.num_envs, row,
                     None if mask is None else mask.data_ptr(), nat.stream_handle())

    def save_snapshot(self, path: str) -> None:
        """On-disk StateSnapshot: little-endian raw arrays + JSON header."""
        import os

        os.makedirs(path, exist_ok=True)
        header = {"layout_hash": self.layout_hash, "fields": {}}
        for k in self.STATE_FIELDS:
            a = getattr(self, k).cpu().numpy()
            a.astype(a.dtype.newbyteorder("<")).tofile(os.path.join(path, f"{k}.bin"))
            header["fields"][k] = {"shape": list(a.shape), "dtype": a.dtype.str}
        with open(os.path.join(path, "manifest.json"), "w") as f:
            json.dump(header, f, indent=1, sort_keys=True)

    def load_snapshot(self, path: str) -> dict:
        import os

        with open(os.path.join(path, "manifest.json")) as f:
            header = json.load(f)
        snap = {"layout_hash": header["layout_hash"]}
        for k, meta in header["fields"].items():
            a = np.fromfile(os.path.join(path, f"{k}.bin"), dtype=np.dtype(meta["dtype"])).reshape(meta["shape"])
            snap[k] = torch.as_tensor(a, device=self.device)
        return snap

    # ------------------------------------------------------------------ views
    def view(self, path: str):
        """Resolve 'art', 'art/link', 'art/joint' or 'actor' into a cached batched view."""
        if path in self._views:
            return self._views[path]
        v = _resolve_view(self, path)
        self._views[path] = v
        return v


def _nearest(name, names):
    import difflib

    return difflib.get_close_matches(name, names, n=3, cutoff=0.3)


class ArticulationView:
    def __init__(self, scene, name, dof_idx):
        self.scene, self.name, self._dof = scene, name, dof_idx  # (N, k) dof index or -1

    def qpos(self):
        return _gather(self.scene.qpos, self._dof)

    def qvel(self):
        return _gather(self.scene.qvel, self._dof)


class JointView(ArticulationView):
    pass


class LinkView:
    def __init__(self, scene, name, link_idx):
        self.scene, self.name, self._link = scene, name, link_idx  # (N,) or -1 where absent

    def pose(self):
        from .pose import PoseBatch

        idx = self._link.clamp(min=0).long()
        rows = self.scene.link_pose[torch.arange(self.scene.num_envs, device=idx.device), idx]
        rows = torch.where((self._link >= 0)[:, None], rows, torch.tensor([0, 0, 0, 1.0, 0, 0, 0],
                                                                           dtype=rows.dtype, device=rows.device))
        return PoseBatch._wrap(rows[:, :3].contiguous(), rows[:, 3:].contiguous())


class ActorView:
    def __init__(self, scene, name, slot):
        self.scene, self.name, self._slot = scene, name, slot

    def pose(self):
        from .pose import PoseBatch

        idx = self._slot.clamp(min=0).long()
        rows = self.scene.actor_pose[torch.arange(self.scene.num_envs, device=idx.device), idx]
        return PoseBatch._wrap(rows[:, :3].contiguous(), rows[:, 3:].contiguous())

    def velocity(self):
        idx = self._slot.clamp(min=0).long()
        return self.scene.actor_vel[torch.arange(self.scene.num_envs, device=idx.device), idx]


def _gather(buf, idx):
    safe = idx.clamp(min=0).long()
    vals = torch.gather(buf, 1, safe)
    return torch.where(idx >= 0, vals, torch.zeros_like(vals))


def _resolve_view(scene: SceneBatch, path: str):
    N, dev = scene.num_envs, scene.device
    ms = [scene.models[m] for m in scene.model_index]
    parts = path.split("/")
    if len(parts) == 1:
        name = parts[0]
        arts = [[d for d, (_, _, a) in enumerate(m.dofs) if a == name] for m in ms]
        if any(m.link_names and any(n.startswith(name + "/") for n in m.link_names) for m in ms):
            k = max(len(a) for a in arts) or 1
            idx = torch.full((N, k), -1, dtype=torch.int32)
            for e, a in enumerate(arts):
                idx[e, :len(a)] = torch.as_tensor(a, dtype=torch.int32)
            return ArticulationView(scene, name, idx.to(dev))
        slots = [m.actor_names.index(name) if name in m.actor_names else -1 for m in ms]
        if any(s >= 0 for s in slots):
            return ActorView(scene, name, torch.as_tensor(slots, dtype=torch.int32, device=dev))
    elif len(parts) == 2:
        links = [m.link_names.index(path) if path in m.link_names else -1 for m in ms]
        if any(l >= 0 for l in links):
            return LinkView(scene, path, torch.as_tensor(links, dtype=torch.int32, device=dev))
        dofs = []
        for m in ms:
            d = -1
            for jn, link in m.joint_names:
                if jn == path:
                    d = m.links[link]["dof"]
            dofs.append(d)
        if any(d >= 0 for d in dofs):
            return JointView(scene, path, torch.as_tensor(dofs, dtype=torch.int32, device=dev)[:, None])
    names = sorted(set(n for m in ms for n in (m.link_names + [j for j, _ in m.joint_names] + m.actor_names)))
    raise ViewLookupError(f"no entity {path!r}; nearest: {_nearest(path, names)}")


def build_batch(descriptors, seed: int = 0, control: ControlSpec = ControlSpec(), device=None,
                shard=None) -> SceneBatch:
    """SPEC.md:186-194.  `shard=(rank, world)` keeps the contiguous global env range
    [rank*N/world, (rank+1)*N/world) with layout maxima taken over ALL envs."""
    descriptors = list(descriptors)
    if shard is None:
        return SceneBatch(descriptors, control, device)
    rank, world = shard
    n = len(descriptors)
    lo, hi = rank * n // world, (rank + 1) * n // world
    return SceneBatch(descriptors[lo:hi], control, device, env_offset=lo, global_descs=descriptors)
