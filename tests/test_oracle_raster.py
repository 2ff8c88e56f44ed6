"""Oracle rasterizer: SPEC render/pointcloud known-answer examples (SPEC.md:465-467, 483-485,
496-500) and the tessellation counts.  CPU only."""

import numpy as np
import pytest

from oracle import raster
from paper_2410_00425_b200 import meshes


def single(kind, size):
    v, f = meshes.shape_mesh(kind, size)
    return {"verts": v, "vert_shape": np.zeros(len(v), np.int32), "tris": f, "tri_shape": np.zeros(len(f), np.int32)}


def frame(mesh, shape_p, cam_p, W=64, H=64, f=None, want_pc=False, seg=7, color=(1.0, 0.5, 0.25)):
    f = H if f is None else f
    return raster.render_frame(mesh, np.array([seg]), np.asarray([shape_p], np.float64), np.array([[1.0, 0, 0, 0]]),
                               np.asarray(cam_p, np.float64), np.array([1.0, 0, 0, 0]), (f, f, W / 2, H / 2), W, H,
                               0.01, 10.0, np.array([color], np.float32), np.array([0.0, 0.0, -1.0]), 0.3, 0.7,
                               (0.0, 0.0, 0.0), want_pc)


@pytest.mark.parametrize("kind,size,tris", [("sphere", (0.1,), 320), ("box", (0.1, 0.2, 0.3), 12),
                                            ("capsule", (0.05, 0.2), 512), ("cylinder", (0.05, 0.2), 64)])
def test_tessellation_counts_closed_outward(kind, size, tris):
    v, f = meshes.shape_mesh(kind, size)
    assert len(f) == tris
    a, b, c = (v[f[:, i]].astype(np.float64) for i in range(3))
    n = np.cross(b - a, c - a)
    assert (np.einsum("ij,ij->i", n, (a + b + c) / 3) > 0).all(), "outward CCW winding"
    edges = {}
    for t in f:
        for i in range(3):
            edges[(t[i], t[(i + 1) % 3])] = edges.get((t[i], t[(i + 1) % 3]), 0) + 1
    assert all(edges.get((j, i), 0) == 1 for (i, j) in edges), "closed manifold"


def test_box_face_on_depth_and_seg():
    # unit box, face-on camera at 2 m, fx=fy=H -> centre depth 1.5 m (1e-3);
    # centre seg = the box's entity id, corner seg = 0
    rgb, depth, seg, _, _ = frame(single("box", (0.5, 0.5, 0.5)), (0, 0, 0), (0, 0, -2.0))
    assert abs(depth[32, 32] - 1.5) < 1e-3
    assert seg[32, 32] == 7 and seg[0, 0] == 0 and depth[0, 0] == 0
    # face-on lit face: intensity 1 -> colour quantised exactly
    assert tuple(rgb[32, 32]) == (255, 128, 64)
    # seg != 0 <=> depth != 0
    assert np.array_equal(seg != 0, depth != 0)
    # coverage: 1 m at 1.5 m with f = 64 px -> ~42.7 px wide
    assert 40 <= (seg[32] != 0).sum() <= 44


def test_wall_back_projection():
    # flat wall normal to the view axis at 2 m -> all points z ~ 2 (1e-3), camera frame
    _, depth, seg, pc, _ = frame(single("box", (5.0, 5.0, 0.1)), (0, 0, 2.1), (0, 0, 0), want_pc=True)
    assert (seg != 0).all()
    assert np.abs(pc[:, 2] - 2.0).max() < 1e-3
    # round trip: back-projected points re-project onto their own pixel centres (0.5 px)
    W = H = 64
    u = pc[:, 0] * 64 / pc[:, 2] + W / 2
    v = pc[:, 1] * 64 / pc[:, 2] + H / 2
    px = np.arange(W * H) % W + 0.5
    py = np.arange(W * H) // W + 0.5
    assert np.abs(u - px).max() < 0.5 and np.abs(v - py).max() < 0.5


def test_empty_scene_renders_background_and_empty_cloud():
    rgb, depth, seg, pc, _ = frame(single("box", (0.1, 0.1, 0.1)), (0, 0, -5.0), (0, 0, 0), want_pc=True)
    assert (seg == 0).all() and (depth == 0).all() and (rgb == 0).all() and (pc == 0).all()


def test_nearest_wins_and_ties_to_lower_triangle():
    # two boxes one behind the other: the nearer one owns the overlap
    m1, m2 = single("box", (0.3, 0.3, 0.3)), single("box", (0.6, 0.6, 0.1))
    v = np.concatenate([m1["verts"], m2["verts"]])
    mesh = {"verts": v, "vert_shape": np.r_[np.zeros(8, np.int32), np.ones(8, np.int32)],
            "tris": np.concatenate([m1["tris"], m2["tris"] + 8]),
            "tri_shape": np.r_[np.zeros(12, np.int32), np.ones(12, np.int32)]}
    rgb, depth, seg, _, _ = raster.render_frame(
        mesh, np.array([3, 9]), np.array([[0, 0, 0.0], [0, 0, 1.0]]), np.tile([1.0, 0, 0, 0], (2, 1)),
        np.array([0, 0, -2.0]), np.array([1.0, 0, 0, 0]), (64, 64, 32, 32), 64, 64, 0.01, 10.0,
        np.ones((2, 3), np.float32), np.array([0, 0, -1.0]), 0.3, 0.7, (0, 0, 0))
    assert seg[32, 32] == 3 and abs(depth[32, 32] - 1.7) < 1e-3
    assert seg[32, 20] == 9 and abs(depth[32, 20] - 2.9) < 1e-3


def test_voxelize_kats():
    # empty cloud -> empty grid; occupancy == brute-force binning
    assert raster.voxelize(np.zeros((0, 3)), None, (0, 0, 0), 0.1, (4, 4, 4)).sum() == 0
    rng = np.random.default_rng(0)
    pts = rng.uniform(-0.1, 0.5, (500, 3)).astype(np.float32)
    g = raster.voxelize(pts, None, (0.0, 0.0, 0.0), 0.1, (4, 4, 4))
    want = np.zeros((4, 4, 4), np.uint8)
    for p in pts:
        i = np.floor(p / np.float32(0.1)).astype(int)
        if (i >= 0).all() and (i < 4).all():
            want[tuple(i)] = 1
    assert np.array_equal(g, want)


def test_greenscreen_kats():
    # empty scene -> background; full cover -> rendered; provenance == seg mask
    rng = np.random.default_rng(1)
    bg = rng.integers(0, 256, (8, 8, 3), dtype=np.uint8)
    rgb = rng.integers(0, 256, (8, 8, 3), dtype=np.uint8)
    assert np.array_equal(raster.composite_greenscreen(rgb, np.zeros((8, 8)), bg), bg)
    assert np.array_equal(raster.composite_greenscreen(rgb, np.ones((8, 8)), bg), rgb)
    seg = np.zeros((8, 8))
    seg[:, :4] = 3
    out = raster.composite_greenscreen(rgb, seg, bg)
    assert np.array_equal(out[:, :4], rgb[:, :4]) and np.array_equal(out[:, 4:], bg[:, 4:])


def test_u8_unit_division_free_form_matches_numpy():
    """csrc/raster.cu u8_unit: c * (1/255) plus one residual correction, each op rounded in
    float32, equals numpy's float32 c / 255 for every c in [0, 255] (the pointcloud colours)."""
    c = np.arange(256, dtype=np.float32)
    k = np.float32(1) / np.float32(255)
    b = c * k
    got = b + (c - b * np.float32(255)) * k
    assert np.array_equal(got.view(np.uint32), (c / np.float32(255)).view(np.uint32))
