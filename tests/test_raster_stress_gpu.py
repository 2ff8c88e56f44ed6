"""Randomised rasterizer stress test: GPU frames vs the CPU oracle rasterizer, bit for bit.

The env tests render the default tabletop view.  This one draws random look-at cameras per
env -- close-ups where one triangle spans most of the frame, grazing views of the ground,
far views where everything is a few pixels -- at odd resolutions (widths that are not a
multiple of 4 take the scalar resolve, non-square frames, frames wider than one tile) and
replays them with every tile size, so every raster path (tiny per-pixel boxes, exact row
spans drawn in-lane, queued long spans, multi-tile frames) is compared against
oracle/raster.py.  Bars: seg, depth bits and rgb identical; pointcloud within 1e-6 (relative above 1 m), as in
test_render_gpu.py.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _look_at_q(eye, target):
    from paper_2410_00425_b200.cameras import look_at

    return np.asarray(look_at(tuple(eye), tuple(target)), np.float64)


def _oracle_frames(env, g, want_pc):
    from oracle import raster
    from oracle.contacts import shape_world_poses
    from oracle.model import Model
    from paper_2410_00425_b200.descriptors import pickcube_desc

    scene, R = env.scene, env.renderer
    model = Model(pickcube_desc(env.spec))
    lp = scene.link_pose.cpu().numpy()
    ap = scene.actor_pose.cpu().numpy()
    SP, SQ = shape_world_poses(model, lp[..., :3], lp[..., 3:], ap[..., :3], ap[..., 3:])
    pose, intr = g["pose"].cpu().numpy(), g["intr"].cpu().numpy()
    out = {}
    for e in range(scene.num_envs):
        for c, cam in enumerate(g["cams"]):
            out[e, c] = raster.render_frame(R.mesh.per_model[0], model.s_seg, SP[e], SQ[e], pose[e, c, :3],
                                            pose[e, c, 3:], intr[e, c], cam.width, cam.height, cam.near, cam.far,
                                            model.s_color[:, :3].astype(np.float32), R.light, R.params.ambient,
                                            R.params.diffuse, R.params.background, want_pc)
    return out


def _random_views(rng, n):
    """(n, 7) camera->world poses: distance 0.08-3 m around the arm/cube, elevation from grazing
    (just above the ground) to top-down."""
    out = np.zeros((n, 7))
    for e in range(n):
        target = np.array([rng.uniform(-0.5, 0.1), rng.uniform(-0.2, 0.2), rng.uniform(0.0, 0.3)])
        dist = math.exp(rng.uniform(math.log(0.08), math.log(3.0)))
        az, el = rng.uniform(-math.pi, math.pi), rng.uniform(0.02, 1.5)
        eye = target + dist * np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
        eye[2] = max(eye[2], 0.02)
        out[e, :3] = eye
        out[e, 3:] = _look_at_q(eye, target)
    return out


@pytest.mark.parametrize("res,obs_mode", [((128, 128), "rgbd"), ((97, 61), "rgbd"), ((200, 150), "pointcloud"),
                                          ((300, 90), "rgbd")])
def test_random_views_all_tiles_bit_exact(cuda, res, obs_mode):
    from paper_2410_00425_b200.cameras import CameraConfig, pinhole
    from paper_2410_00425_b200.tasks import make_task

    w, h = res
    N = 12
    cams = [CameraConfig("cam", pose_p=(0.3, 0.3, 0.3), pose_q=tuple(_look_at_q((0.3, 0.3, 0.3), (0, 0, 0))),
                         **pinhole(w, h, 60.0))]
    env = make_task("PickCube", N, seed=11, obs_mode=obs_mode, cameras=cams)
    env.reset(seed=11)
    for t in range(3):
        env.step_random(t)
    rng = np.random.default_rng(w * 1000 + h)
    g = env.renderer.groups[0]
    views = _random_views(rng, N)
    g["pose"].copy_(torch.as_tensor(views[:, None, :], device=g["pose"].device))
    # random focal lengths too (wide to telephoto)
    f = rng.uniform(0.3, 3.0, N) * w / 2
    intr = np.stack([f, f * rng.uniform(0.8, 1.25, N), rng.uniform(0.3, 0.7, N) * w, rng.uniform(0.3, 0.7, N) * h], -1)
    g["intr"].copy_(torch.as_tensor(intr[:, None, :].astype(np.float32), device=g["intr"].device))
    want_pc = obs_mode == "pointcloud"
    want = _oracle_frames(env, g, want_pc)
    hit_counts = []
    # every tile size, twice: work queues hand out spans in a different order on every launch
    for tile in (0, 32, 64, 128, 256, 0, 32, 64, 128, 256):
        env.renderer.c_params.tile = tile
        for k in ("rgb", "depth", "seg"):
            g[k].zero_()
        env.renderer.render()
        torch.cuda.synchronize()
        rgb, depth, seg = g["rgb"].cpu().numpy(), g["depth"].cpu().numpy(), g["seg"].cpu().numpy()
        pc = g["pc"].cpu().numpy() if want_pc else None
        for e in range(N):
            w_rgb, w_depth, w_seg, w_pc, _ = want[e, 0]
            assert np.array_equal(seg[e, 0].view(np.uint16), w_seg), f"tile {tile} env {e}: seg"
            assert np.array_equal(depth[e, 0].view(np.uint32), w_depth.view(np.uint32)), f"tile {tile} env {e}: depth"
            assert np.array_equal(rgb[e, 0], w_rgb), f"tile {tile} env {e}: rgb"
            if want_pc:
                assert np.abs(pc[e, 0] - w_pc).max() <= 1e-6 * max(1.0, float(np.abs(w_pc).max())), f"tile {tile} env {e}: pc"
            hit_counts.append(int((w_seg != 0).sum()))
    # the random views are not all empty: most frames see something, some are mostly covered
    assert np.mean(np.asarray(hit_counts) > 0) > 0.5 and max(hit_counts) > 0.5 * w * h


@pytest.mark.parametrize("caps,obs_mode", [("4,16", "rgbd"), ("1,1", "pointcloud"), ("256,64", "rgbd")])
def test_overflow_paths_bit_exact(cuda, caps, obs_mode):
    """With the big-record and span capacities lowered (BS_RENDER_CAPS, a test knob read once per
    process), triangles past the record capacity are set up in later rounds (at most the record
    capacity per round) and row items run in windows of the span capacity -- "1,1" makes every
    big triangle its own round and every row its own window.  Frames must equal the oracle."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "raster_caps_child.py"), obs_mode],
                       env=dict(os.environ, BS_RENDER_CAPS=caps), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("near,far", [(0.3, 0.9), (0.01, 0.45)])
def test_near_far_planes_and_close_ups_bit_exact(cuda, near, far):
    """Depth-range edge cases: a far plane that cuts through the scene (fragments beyond it are
    dropped per pixel) and cameras so close that vertices fall behind the near plane or outside
    the guard band (whole triangles culled) -- every pixel equals the oracle's."""
    from paper_2410_00425_b200.cameras import CameraConfig, pinhole
    from paper_2410_00425_b200.tasks import make_task

    w = h = 96
    N = 8
    cams = [CameraConfig("cam", pose_p=(0.3, 0.3, 0.3), pose_q=tuple(_look_at_q((0.3, 0.3, 0.3), (0, 0, 0))),
                         near=near, far=far, **pinhole(w, h, 60.0))]
    env = make_task("PickCube", N, seed=2, obs_mode="rgbd", cameras=cams)
    env.step_random(0)
    g = env.renderer.groups[0]
    rng = np.random.default_rng(int(far * 1000))
    views = np.zeros((N, 7))
    cube = env.scene.actor_pose.cpu().numpy()[:, 0, :3]
    for e in range(N):  # from just outside the cube to a grazing view along the ground
        target = cube[e] + rng.uniform(-0.02, 0.02, 3)
        d = [0.012, 0.02, 0.05, 0.3, 0.6, 1.0, 0.04, 0.25][e]
        az = rng.uniform(-np.pi, np.pi)
        eye = target + d * np.array([np.cos(az), np.sin(az), 0.4 if e < 6 else 0.05])
        eye[2] = max(eye[2], 0.005)
        views[e, :3], views[e, 3:] = eye, _look_at_q(eye, target)
    g["pose"].copy_(torch.as_tensor(views[:, None, :], device=g["pose"].device))
    want = _oracle_frames(env, g, False)
    env.renderer.render()
    torch.cuda.synchronize()
    rgb, depth, seg = g["rgb"].cpu().numpy(), g["depth"].cpu().numpy(), g["seg"].cpu().numpy()
    clipped = 0
    for e in range(N):
        w_rgb, w_depth, w_seg, _, _ = want[e, 0]
        assert np.array_equal(seg[e, 0].view(np.uint16), w_seg), f"env {e}: seg"
        assert np.array_equal(depth[e, 0].view(np.uint32), w_depth.view(np.uint32)), f"env {e}: depth"
        assert np.array_equal(rgb[e, 0], w_rgb), f"env {e}: rgb"
        hit = w_depth[w_depth > 0]
        assert hit.size == 0 or (hit.min() >= near and hit.max() <= far)
        clipped += int((w_depth == 0).sum())
    assert clipped > 0  # the far plane / near plane actually removed something
