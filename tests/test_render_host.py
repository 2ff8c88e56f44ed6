"""Host-side render logic (no GPU): camera randomisation properties."""

import numpy as np


def test_randomize_cameras_properties():
    from paper_2410_00425_b200.cameras import CameraJitter, default_cameras, randomize_cameras

    cams = default_cameras()
    p0, k0 = randomize_cameras(cams, 4, 7, CameraJitter())
    assert (p0 == p0[:1]).all() and (k0 == k0[:1]).all()  # zero jitter -> identical configs
    j = CameraJitter(pos=0.02, rot=0.035, focal=0.05)
    p1, k1 = randomize_cameras(cams, 4, 7, j)
    p2, k2 = randomize_cameras(cams, 4, 7, j)
    assert np.array_equal(p1, p2) and np.array_equal(k1, k2)  # same seed -> bitwise equal
    assert not np.array_equal(p1[0], p1[1])  # envs differ
    assert np.abs(p1[:, 0, :3] - p0[:, 0, :3]).max() <= 0.02
    # shard-invariant: env 3 of a 4-env draw == env 1 of the shard starting at global env 2
    p3, _ = randomize_cameras(cams, 2, 7, j, env_offset=2)
    assert np.array_equal(p3[1], p1[3])
