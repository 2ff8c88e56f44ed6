"""Cameras for the batched rasterizer (torch-free host code): CameraConfig,
randomize_cameras, render parameters and the default tabletop view."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import hostmath as hm
from . import rng as brng
from .errors import InputError

OBS_MODES = ("state", "rgb", "depth", "rgbd", "rgb+depth", "seg", "rgb+depth+seg", "pointcloud")


@dataclass(frozen=True)
class CameraConfig:
    """SPEC.md:450.  pose = camera -> world (OpenCV: x right, y down, z forward) or, when
    `mount` names a link, the camera's offset in that link's frame."""

    name: str = "cam"
    width: int = 128
    height: int = 128
    fx: float = 110.85
    fy: float = 110.85
    cx: float = 64.0
    cy: float = 64.0
    pose_p: tuple = (0.0, 0.0, 1.0)
    pose_q: tuple = (1.0, 0.0, 0.0, 0.0)
    mount: str = None
    near: float = 0.01
    far: float = 10.0

    def __post_init__(self):
        if not (0.0 < self.near < self.far):
            raise InputError(f"camera {self.name!r}: need 0 < near < far")
        if self.width < 1 or self.height < 1:
            raise InputError(f"camera {self.name!r}: width and height must be >= 1")


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """Camera -> world quaternion for an OpenCV camera at `eye` looking at `target`."""
    return tuple(hm.look_at(eye, target, up)[1])


def pinhole(width, height, fov_y_deg):
    fy = (height / 2.0) / math.tan(math.radians(fov_y_deg) / 2.0)
    return dict(width=width, height=height, fx=fy, fy=fy, cx=width / 2.0, cy=height / 2.0)


def default_cameras(width=128, height=128):
    """PickCube-style tabletop view (BASELINE configs C3/C4: one 128x128 camera)."""
    eye, target = (0.15, 0.5, 0.4), (-0.15, 0.0, 0.02)
    return [CameraConfig("base_camera", pose_p=eye, pose_q=look_at(eye, target), **pinhole(width, height, 60.0))]


@dataclass(frozen=True)
class CameraJitter:
    """randomize_cameras ranges: uniform +-pos (m), +-rot (rad, about a
    uniformly drawn axis-angle vector's components), +-focal (fraction of fx/fy)."""

    pos: float = 0.0
    rot: float = 0.0
    focal: float = 0.0


def randomize_cameras(cameras, num_envs, seed, jitter: CameraJitter, env_offset=0):
    """Per-env camera poses/intrinsics (N, C, 7) f64 and (N, C, 4) f32, drawn from each env's
    Philox stream (counter = (camera, 0, global env, 'CAMR')); zero jitter -> the base config
    for every env, bitwise."""
    C = len(cameras)
    ids = np.arange(env_offset, env_offset + num_envs, dtype=np.uint64)
    pose = np.zeros((num_envs, C, 7))
    intr = np.zeros((num_envs, C, 4), np.float32)
    for c, cam in enumerate(cameras):
        base_p = np.asarray(cam.pose_p, np.float64)
        base_q = hm.qnormalize(cam.pose_q)
        pose[:, c, :3] = base_p
        pose[:, c, 3:] = base_q
        intr[:, c] = (cam.fx, cam.fy, cam.cx, cam.cy)
        if jitter.pos or jitter.rot or jitter.focal:
            u = brng.uniforms(seed, ids, c, brng.TAG_CAMERA, 8)   # (N, 8) in [0, 1)
            pose[:, c, :3] = base_p + jitter.pos * (2.0 * u[:, 0:3] - 1.0)
            rv = jitter.rot * (2.0 * u[:, 3:6] - 1.0)
            for e in range(num_envs):
                ang = float(np.linalg.norm(rv[e]))
                if ang > 0.0:
                    ax = rv[e] / ang
                    dq = np.array([math.cos(ang / 2), *(ax * math.sin(ang / 2))])
                    pose[e, c, 3:] = hm.qnormalize(hm.qmul(base_q, dq))
            s = 1.0 + jitter.focal * (2.0 * u[:, 6] - 1.0)
            intr[:, c, 0] = (cam.fx * s).astype(np.float32)
            intr[:, c, 1] = (cam.fy * s).astype(np.float32)
    return pose, intr


@dataclass
class RenderParams:
    light_dir: tuple = (0.35, 0.25, 1.0)   # towards the light, world frame (normalised)
    ambient: float = 0.35
    diffuse: float = 0.65
    background: tuple = (0.0, 0.0, 0.0)
    tile: int = 128
