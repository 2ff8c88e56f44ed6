"""Repeated renders of random views vs the oracle (order-dependent raster bugs show up as sporadic
bad frames).  Usage: python tools/raster_probe.py [reps] [tile]"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import test_raster_stress_gpu as T
from paper_2410_00425_b200.cameras import CameraConfig, pinhole
from paper_2410_00425_b200.tasks import make_task
w, h = 128, 128
N = 12
cams = [CameraConfig("cam", pose_p=(0.3, 0.3, 0.3), pose_q=tuple(T._look_at_q((0.3, 0.3, 0.3), (0, 0, 0))), **pinhole(w, h, 60.0))]
env = make_task("PickCube", N, seed=11, obs_mode="rgbd", cameras=cams)
env.reset(seed=11)
for t in range(3):
    env.step_random(t)
rng = np.random.default_rng(w * 1000 + h)
g = env.renderer.groups[0]
views = T._random_views(rng, N)
g["pose"].copy_(torch.as_tensor(views[:, None, :], device=g["pose"].device))
f = rng.uniform(0.3, 3.0, N) * w / 2
intr = np.stack([f, f * rng.uniform(0.8, 1.25, N), rng.uniform(0.3, 0.7, N) * w, rng.uniform(0.3, 0.7, N) * h], -1)
g["intr"].copy_(torch.as_tensor(intr[:, None, :].astype(np.float32), device=g["intr"].device))
want = T._oracle_frames(env, g, False)
from oracle.contacts import shape_world_poses
from oracle.model import Model
from oracle import se3
from paper_2410_00425_b200.descriptors import pickcube_desc
model = Model(pickcube_desc(env.spec))
lp = env.scene.link_pose.cpu().numpy(); ap = env.scene.actor_pose.cpu().numpy()
SP, SQ = shape_world_poses(model, lp[..., :3], lp[..., 3:], ap[..., :3], ap[..., 3:])
mesh = env.renderer.mesh.per_model[0]
pose_np, intr_np = g["pose"].cpu().numpy(), g["intr"].cpu().numpy()
def tri_box(e, t):
    F = np.float32
    pcw, qcw = se3.inverse(pose_np[e, 0, :3][None], pose_np[e, 0, 3:][None])
    S = SP.shape[1]
    pcs, qcs = se3.compose(np.broadcast_to(pcw, (S, 3)), np.broadcast_to(qcw, (S, 4)), SP[e], SQ[e])
    R = se3.qmat(qcs).astype(F); tt = pcs.astype(F)
    fx, fy, cx, cy = (F(x) for x in intr_np[e, 0])
    X = []
    for vi in mesh["tris"][t]:
        v = mesh["verts"][vi].astype(F); sh = mesh["vert_shape"][vi]
        xc = np.array([((R[sh][i, 0] * v[0] + R[sh][i, 1] * v[1]) + R[sh][i, 2] * v[2]) + tt[sh][i] for i in range(3)], F)
        X.append(((fx * xc[0]) / xc[2] + cx, (fy * xc[1]) / xc[2] + cy))
    X = np.array(X)
    return X.min(0), X.max(0)
bad = 0
env.renderer.c_params.tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    env.renderer.render()
    torch.cuda.synchronize()
    seg = g["seg"].cpu().numpy()
    for e in range(N):
        d = (seg[e, 0].view(np.uint16) != want[e, 0][2])
        if d.any():
            bad += 1
            ys, xs = np.nonzero(d)
            kb = want[e, 0][4].reshape(h, w)[ys[0], xs[0]]
            t = int(kb & np.uint64(0xffffffff))
            print("rep", rep, "env", e, "bad px", d.sum(), "at", list(zip(ys[:5], xs[:5])), "got", seg[e,0].view(np.uint16)[ys[0], xs[0]], "want", want[e,0][2][ys[0], xs[0]], "tri", t, "depth", g["depth"][e,0,ys[0],xs[0]].item(), "want depth", want[e,0][1][ys[0], xs[0]], "box", tri_box(e, t))
print("bad frames", bad)
# triangle box sizes of the failing winners (oracle projection)
