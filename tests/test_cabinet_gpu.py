"""GPU OpenCabinet (heterogeneous articulated objects, BASELINE config 4) vs the CPU oracle.

Per-env cabinets with 2-6 drawers/doors give up to 2^2 + ... + 2^6 distinct layouts in one batch
(SPEC.md:174-177, 615).  Bars: target joints and reset state bit-exact; integer flags
bit-exact; one-step float state within 1e-9 from an identical start state; the rendered
pointcloud of a heterogeneous scene bit-matches the oracle rasterizer.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, SEED = 8, 2


@pytest.fixture(scope="module")
def pair(cuda):
    from oracle.tasks import OpenCabinetOracle
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("OpenCabinet", N, seed=SEED)
    orc = OpenCabinetOracle(env.spec, env.descs, SEED)
    return env, orc


def test_heterogeneous_layouts_and_reset(pair):
    env, orc = pair
    assert len(env.scene.models) > 1
    dofs = [env.scene.models[m].D for m in env.scene.model_index]
    assert min(dofs) >= 5 and max(dofs) <= 9
    assert np.array_equal(env.scene.target_dof.cpu().numpy(), orc.target)
    snap = orc.snapshot()
    q = env.scene.qpos.cpu().numpy()
    assert np.array_equal(q, snap["q"])


def test_one_step_parity(pair):
    from oracle.philox import action_uniforms
    from paper_2410_00425_b200 import _native as nat

    env, orc = pair
    for t in range(12):
        q0, qd0 = env.scene.qpos.cpu().numpy(), env.scene.qvel.cpu().numpy()
        orc.load(q0, qd0)
        orc.elapsed[:] = env.scene.elapsed.cpu().numpy()
        orc.reset_count[:] = env.scene.reset_count.cpu().numpy().astype(np.uint64)
        orc.target[:] = env.scene.target_dof.cpu().numpy()
        a = torch.empty((N, 3), dtype=torch.float32, device=env.device)
        nat.call("bs_random_actions", SEED, t, 0, N, 3, a.data_ptr(), nat.stream_handle())
        r = env.step(a)
        o_rew, o_term, o_trunc, o_info, _ = orc.step(action_uniforms(SEED, t, np.arange(N), 3))
        assert np.array_equal(r.terminated.cpu().numpy().astype(bool), o_term), t
        assert np.array_equal(r.truncated.cpu().numpy().astype(bool), o_trunc), t
        assert np.array_equal(r.info["success"].cpu().numpy().astype(bool), o_info["success"]), t
        assert np.abs(r.reward.cpu().numpy() - o_rew).max() < 1e-5
        snap = orc.snapshot()
        assert np.abs(env.scene.qpos.cpu().numpy() - snap["q"]).max() < 1e-9, t
        assert np.abs(env.scene.qvel.cpu().numpy() - snap["qd"]).max() < 1e-9, t


def test_state_obs_layout(pair):
    env, _ = pair
    obs = env.reset(seed=SEED)
    D = env.scene.D_max
    assert obs.shape == (N, 2 * D + 3 + 13 * env.scene.A_max + 3)
    ee = obs[:, 2 * D:2 * D + 3].cpu().numpy()
    lp = env.scene.link_pose.cpu().numpy()
    idx = env.scene.models[0].link_names.index("arm/ee")
    assert np.abs(ee - lp[:, idx, :3]).max() < 1e-6


def test_pointcloud_heterogeneous(cuda):
    from oracle import raster
    from oracle.contacts import shape_world_poses
    from oracle.model import Model
    from paper_2410_00425_b200.tasks import make_task

    env = make_task("OpenCabinet", 4, seed=5, obs_mode="pointcloud")
    env.step_random(0)
    torch.cuda.synchronize()
    R = env.renderer
    g = R.groups[0]
    cam = g["cams"][0]
    pc = g["pc"].cpu().numpy()[:, 0]
    lp = env.scene.link_pose.cpu().numpy()
    pose, intr = g["pose"].cpu().numpy(), g["intr"].cpu().numpy()
    for e in range(4):
        mi = env.scene.model_index[e]
        model = Model(env.descs[e])
        L = model.L
        SP, SQ = shape_world_poses(model, lp[e:e + 1, :L, :3], lp[e:e + 1, :L, 3:], np.zeros((1, 0, 3)),
                                   np.zeros((1, 0, 4)))
        rgb, depth, seg, wpc, _ = raster.render_frame(
            R.mesh.per_model[mi], model.s_seg, SP[0], SQ[0], pose[e, 0, :3], pose[e, 0, 3:], intr[e, 0], cam.width,
            cam.height, cam.near, cam.far, model.s_color[:, :3].astype(np.float32), R.light, R.params.ambient,
            R.params.diffuse, R.params.background, True)
        assert np.array_equal(g["seg"][e, 0].cpu().numpy().view(np.uint16), seg), e
        assert np.abs(pc[e] - wpc).max() <= 1e-6, e
