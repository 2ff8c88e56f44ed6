"""GPU PickHetero (heterogeneous scenes, BASELINE config 5) vs the CPU oracle.

Every env has its own object kind/size (sphere / box / capsule, resting pose per A-26), its
own colour (texture randomisation) and its own jittered cameras (2 x 256x256).  Bars: reset
state exact; one-step state within 1e-9 from identical starts; integer flags bit-exact;
frames from both cameras bit-exact against the oracle rasterizer.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, SEED = 8, 4


def gpu_snapshot(env):
    s = env.scene
    ap, av = s.actor_pose.cpu().numpy(), s.actor_vel.cpu().numpy()
    return {"q": s.qpos.cpu().numpy()[:, :3], "qd": s.qvel.cpu().numpy()[:, :3], "ap": ap[:, :, :3],
            "aq": ap[:, :, 3:], "av": av[:, :, :3], "aw": av[:, :, 3:], "goal": s.goal.cpu().numpy(),
            "elapsed": s.elapsed.cpu().numpy()}


def test_state_parity(cuda):
    from oracle.philox import action_uniforms
    from oracle.tasks import PickHeteroOracle
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickHetero", N, seed=SEED)
    kinds = {m.desc.actors[0].kind for m in env.scene.models}
    assert len(env.scene.models) > 2 and len(kinds) >= 2
    orc = PickHeteroOracle(env.spec, env.descs, SEED)
    g, o = gpu_snapshot(env), orc.snapshot()
    for k in ("q", "ap", "goal"):
        assert np.array_equal(g[k], o[k]), k
    assert np.abs(g["aq"] - o["aq"]).max() <= 1e-15  # device sincos vs libm: <= 1 ulp
    for t in range(12):
        orc.load(gpu_snapshot(env), env.scene.reset_count.cpu().numpy().astype(np.uint64))
        r = env.step_random(t)
        o_rew, o_term, o_trunc, o_info = orc.step(action_uniforms(SEED, t, np.arange(N), 3))
        assert np.array_equal(r.terminated.cpu().numpy().astype(bool), o_term), t
        assert np.array_equal(r.truncated.cpu().numpy().astype(bool), o_trunc), t
        g, o = gpu_snapshot(env), orc.snapshot()
        for k in ("q", "qd", "ap", "aq", "av", "aw"):
            assert np.abs(g[k] - o[k]).max() < 1e-9, (t, k)


def test_two_jittered_cameras_bit_exact(cuda):
    from oracle import raster
    from oracle.contacts import shape_world_poses
    from oracle.model import Model
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("PickHetero", 3, seed=SEED, obs_mode="rgbd")
    env.step_random(0)
    torch.cuda.synchronize()
    R = env.renderer
    assert len(R.groups) == 1 and len(R.groups[0]["cams"]) == 2
    g = R.groups[0]
    pose, intr = g["pose"].cpu().numpy(), g["intr"].cpu().numpy()
    assert not np.array_equal(pose[0, 0], pose[1, 0])  # per-env camera jitter
    colors = R.env_color.cpu().numpy()
    lp, ap = env.scene.link_pose.cpu().numpy(), env.scene.actor_pose.cpu().numpy()
    for e in range(3):
        model = Model(env.descs[e])
        SP, SQ = shape_world_poses(model, lp[e:e + 1, :model.L, :3], lp[e:e + 1, :model.L, 3:],
                                   ap[e:e + 1, :, :3], ap[e:e + 1, :, 3:])
        mi = env.scene.model_index[e]
        for c, cam in enumerate(g["cams"]):
            rgb, depth, seg, _, _ = raster.render_frame(
                R.mesh.per_model[mi], model.s_seg, SP[0], SQ[0], pose[e, c, :3], pose[e, c, 3:], intr[e, c],
                cam.width, cam.height, cam.near, cam.far, colors[e, :model.S], R.light, R.params.ambient,
                R.params.diffuse, R.params.background)
            assert np.array_equal(g["seg"][e, c].cpu().numpy().view(np.uint16), seg), (e, c)
            assert np.array_equal(g["depth"][e, c].cpu().numpy().view(np.uint32), depth.view(np.uint32)), (e, c)
            assert np.array_equal(g["rgb"][e, c].cpu().numpy(), rgb), (e, c)
