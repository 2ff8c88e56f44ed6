"""Child process of test_raster_stress_gpu.py::test_overflow_paths_bit_exact: renders random
views with the record / span capacities lowered through BS_RENDER_CAPS (read once per process)
and exits non-zero on any mismatch against the oracle rasterizer."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import test_raster_stress_gpu as T  # noqa: E402


def main():
    from paper_2410_00425_b200.cameras import CameraConfig, pinhole
    from paper_2410_00425_b200.tasks import make_task

    w, h, N = 128, 96, 8
    obs_mode = sys.argv[1] if len(sys.argv) > 1 else "rgbd"
    cams = [CameraConfig("cam", pose_p=(0.3, 0.3, 0.3), pose_q=tuple(T._look_at_q((0.3, 0.3, 0.3), (0, 0, 0))),
                         **pinhole(w, h, 60.0))]
    env = make_task("PickCube", N, seed=5, obs_mode=obs_mode, cameras=cams)
    env.step_random(0)
    rng = np.random.default_rng(7)
    g = env.renderer.groups[0]
    g["pose"].copy_(torch.as_tensor(T._random_views(rng, N)[:, None, :], device=g["pose"].device))
    want = T._oracle_frames(env, g, obs_mode == "pointcloud")
    bad = 0
    for tile in (0, 64):
        env.renderer.c_params.tile = tile
        env.renderer.render()
        torch.cuda.synchronize()
        for e in range(N):
            w_rgb, w_depth, w_seg, w_pc, _ = want[e, 0]
            ok = (np.array_equal(g["seg"][e, 0].cpu().numpy().view(np.uint16), w_seg)
                  and np.array_equal(g["depth"][e, 0].cpu().numpy().view(np.uint32), w_depth.view(np.uint32))
                  and np.array_equal(g["rgb"][e, 0].cpu().numpy(), w_rgb))
            if w_pc is not None:
                ok = ok and np.abs(g["pc"][e, 0].cpu().numpy() - w_pc).max() <= 1e-6 * max(1.0, float(np.abs(w_pc).max()))
            bad += not ok
    print("bad frames", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
