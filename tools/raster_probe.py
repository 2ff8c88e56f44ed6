"""Repeated renders of random views against the oracle rasterizer.

Order-dependent rasterizer bugs (work queues hand out spans in a different order on every
launch) show up as sporadic bad frames.  For each bad frame the probe prints the first wrong
pixel, the oracle's winning triangle there and its projected box.

    python tools/raster_probe.py [reps] [tile]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_raster_stress_gpu as T  # noqa: E402
from oracle import se3  # noqa: E402
from oracle.contacts import shape_world_poses  # noqa: E402
from oracle.model import Model  # noqa: E402
from paper_2410_00425_b200.cameras import CameraConfig, pinhole  # noqa: E402
from paper_2410_00425_b200.descriptors import pickcube_desc  # noqa: E402
from paper_2410_00425_b200.tasks import make_task  # noqa: E402

W, H, N = 128, 128, 12
F = np.float32


def build_env():
    eye = (0.3, 0.3, 0.3)
    cams = [CameraConfig("cam", pose_p=eye, pose_q=tuple(T._look_at_q(eye, (0, 0, 0))), **pinhole(W, H, 60.0))]
    env = make_task("PickCube", N, seed=11, obs_mode="rgbd", cameras=cams)
    env.reset(seed=11)
    for t in range(3):
        env.step_random(t)
    rng = np.random.default_rng(W * 1000 + H)
    g = env.renderer.groups[0]
    g["pose"].copy_(torch.as_tensor(T._random_views(rng, N)[:, None, :], device=g["pose"].device))
    f = rng.uniform(0.3, 3.0, N) * W / 2
    intr = np.stack([f, f * rng.uniform(0.8, 1.25, N), rng.uniform(0.3, 0.7, N) * W, rng.uniform(0.3, 0.7, N) * H], -1)
    g["intr"].copy_(torch.as_tensor(intr[:, None, :].astype(np.float32), device=g["intr"].device))
    return env, g


def tri_box(env, g, e, t):
    """Projected pixel box (min, max) of triangle t in env e's frame (oracle arithmetic)."""
    model = Model(pickcube_desc(env.spec))
    lp, ap = env.scene.link_pose.cpu().numpy(), env.scene.actor_pose.cpu().numpy()
    SP, SQ = shape_world_poses(model, lp[..., :3], lp[..., 3:], ap[..., :3], ap[..., 3:])
    pose, intr = g["pose"].cpu().numpy(), g["intr"].cpu().numpy()
    mesh = env.renderer.mesh.per_model[0]
    pcw, qcw = se3.inverse(pose[e, 0, :3][None], pose[e, 0, 3:][None])
    S = SP.shape[1]
    pcs, qcs = se3.compose(np.broadcast_to(pcw, (S, 3)), np.broadcast_to(qcw, (S, 4)), SP[e], SQ[e])
    R, tt = se3.qmat(qcs).astype(F), pcs.astype(F)
    fx, fy, cx, cy = (F(x) for x in intr[e, 0])
    pts = []
    for vi in mesh["tris"][t]:
        v, sh = mesh["verts"][vi].astype(F), mesh["vert_shape"][vi]
        xc = np.array([((R[sh][i, 0] * v[0] + R[sh][i, 1] * v[1]) + R[sh][i, 2] * v[2]) + tt[sh][i] for i in range(3)], F)
        pts.append(((fx * xc[0]) / xc[2] + cx, (fy * xc[1]) / xc[2] + cy))
    pts = np.array(pts)
    return pts.min(0), pts.max(0)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    env, g = build_env()
    env.renderer.c_params.tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    want = T._oracle_frames(env, g, False)
    bad = 0
    for rep in range(reps):
        env.renderer.render()
        torch.cuda.synchronize()
        seg, depth = g["seg"].cpu().numpy(), g["depth"].cpu().numpy()
        for e in range(N):
            wseg = want[e, 0][2]
            diff = seg[e, 0].view(np.uint16) != wseg
            if not diff.any():
                continue
            bad += 1
            ys, xs = np.nonzero(diff)
            y, x = ys[0], xs[0]
            key = want[e, 0][4].reshape(H, W)[y, x]
            t = int(key & np.uint64(0xFFFFFFFF))
            print(f"rep {rep} env {e}: {int(diff.sum())} bad px, first at ({y}, {x}): got seg "
                  f"{seg[e, 0].view(np.uint16)[y, x]} depth {depth[e, 0, y, x]:.6f}, want seg {wseg[y, x]} depth "
                  f"{want[e, 0][1][y, x]:.6f}" + (f" (triangle {t}, box {tri_box(env, g, e, t)})" if key != ~np.uint64(0) else ""))
    print("bad frames", bad)


if __name__ == "__main__":
    main()
