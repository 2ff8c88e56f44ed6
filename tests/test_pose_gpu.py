"""GPU pose kernels vs the reference: bit-exact fp64 for normalize/compose/inverse/matrix
round trip (golden vectors from the reference itself), plus the reference's own
test_pose.py cases replayed through the device PoseBatch (seeds 0-11, same tolerances)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def bits(a):
    """Bit patterns with every NaN mapped to one value: NaN sign/payload is not part of
    the contract (x86 and sm_100a produce different default NaNs); signed zeros are."""
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = a.view(np.uint64).copy()
    b[np.isnan(a)] = 0x7FF8000000000000
    return b


def _explain(got, want):
    g, w = bits(got), bits(want)
    bad = np.argwhere(g != w)
    return f"{len(bad)} mismatches, first at {bad[:3].tolist()}"


@pytest.fixture(scope="module")
def P(cuda):
    from paper_2410_00425_b200 import pose

    return pose


def test_normalize_compose_inverse_bit_exact(P, pose_golden):
    g = pose_golden
    assert np.array_equal(bits(P.quat_normalize(torch.tensor(g["qa_raw"]).cuda())), bits(g["qa_norm"]))
    A = P.PoseBatch(g["pa"], g["qa_raw"])
    B = P.PoseBatch(g["pb"], g["qb_raw"])
    C = A.compose(B)
    assert np.array_equal(bits(C.p), bits(g["compose_p"]))
    assert np.array_equal(bits(C.q), bits(g["compose_q"]))
    I = A.inverse()
    assert np.array_equal(bits(I.p), bits(g["inverse_p"])), _explain(I.p, g["inverse_p"])
    assert np.array_equal(bits(I.q), bits(g["inverse_q"])), _explain(I.q, g["inverse_q"])
    W = A.compose(B).inverse().compose(A.inverse())
    assert np.array_equal(bits(W.p), bits(g["worked_p"]))
    assert np.array_equal(bits(W.q), bits(g["worked_q"]))
    S = A[0]
    assert np.array_equal(bits(S.compose(B).p), bits(g["bcast_left_p"]))
    assert np.array_equal(bits(B.compose(S).q), bits(g["bcast_right_q"]))


def test_matrix_round_trip_bit_exact(P, pose_golden):
    g = pose_golden
    A = P.PoseBatch(g["pa"], g["qa_raw"])
    M = A.to_matrix().matrices
    assert np.array_equal(bits(M), bits(g["to_matrix"]))
    F = P.PoseBatch.from_matrix(g["to_matrix"])
    assert np.array_equal(bits(F.p), bits(g["from_matrix_p"]))
    assert np.array_equal(bits(F.q), bits(g["from_matrix_q"]))


def test_transform_points(P, pose_golden):
    g = pose_golden
    A = P.PoseBatch(g["pa"], g["qa_raw"])
    got = A.transform_points(g["pts"]).cpu().numpy()
    want = g["transform_points"]
    fin = np.isfinite(want)
    assert np.array_equal(fin, np.isfinite(got))
    assert np.abs(got[fin] - want[fin]).max() < 1e-12
    single = A[0].transform_points(g["pts"][0]).cpu().numpy()
    assert np.abs(single - g["transform_points_single"]).max() < 1e-12


def test_chain_bit_exact(P, pose_golden):
    g = pose_golden
    step = P.PoseBatch(g["pa"][:4], g["qa_raw"][:4])
    acc = P.PoseBatch.identity(4)
    for _ in range(1000):
        acc = acc.compose(step)
    assert np.array_equal(bits(acc.p), bits(g["chain_p"]))
    assert np.array_equal(bits(acc.q), bits(g["chain_q"]))


def test_f32_speed_path_tolerance(P, pose_golden):
    g = pose_golden
    n = 1024
    A = P.PoseBatch(g["pa"][:n], g["qa_raw"][:n], dtype=torch.float32)
    B = P.PoseBatch(g["pb"][:n], g["qb_raw"][:n], dtype=torch.float32)
    C = A.compose(B)
    assert np.abs(C.p.double().cpu().numpy() - g["compose_p"][:n]).max() < 5e-6
    assert np.abs(C.q.double().cpu().numpy() - g["compose_q"][:n]).max() < 5e-6


# ---- the reference's own test_pose.py, replayed on the device -------------------------

def random_poses(P, rng, n):
    p = rng.uniform(-2.0, 2.0, size=(n, 3))
    q = rng.normal(size=(n, 4))
    return P.PoseBatch(p, q)


def matrix_oracle(pose):
    p, q = pose.numpy()
    n = len(p)
    out = np.zeros((n, 4, 4))
    for i in range(n):
        w, x, y, z = q[i]
        out[i, :3, :3] = [[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                          [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                          [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]]
        out[i, :3, 3] = p[i]
        out[i, 3, 3] = 1.0
    return out


def test_ref_identity_left_right(P):
    p = random_poses(P, np.random.default_rng(0), 32)
    eye = P.PoseBatch.identity(1)
    assert eye.compose(p).allclose(p, atol=1e-12)
    assert p.compose(eye).allclose(p, atol=1e-12)


def test_ref_inverse_gives_identity(P):
    p = random_poses(P, np.random.default_rng(1), 64)
    ident = p.compose(p.inverse())
    ip, iq = ident.numpy()
    assert np.abs(ip).max() < 1e-9
    assert np.abs(iq - np.array([1.0, 0, 0, 0])).max() < 1e-9


def test_ref_matches_matrix_oracle_bulk(P):
    rng = np.random.default_rng(2)
    a = random_poses(P, rng, 10_000)
    b = random_poses(P, rng, 10_000)
    got = a.compose(b).to_matrix().matrices.cpu().numpy()
    want = matrix_oracle(a) @ matrix_oracle(b)
    assert np.abs(got - want).max() < 1e-9


def test_ref_incompatible_sizes(P):
    from paper_2410_00425_b200.errors import DimensionError

    rng = np.random.default_rng(4)
    with pytest.raises(DimensionError, match="3.*5|5.*3"):
        random_poses(P, rng, 3).compose(random_poses(P, rng, 5))


def test_ref_associativity_and_drift(P):
    rng = np.random.default_rng(5)
    a, b, c = (random_poses(P, rng, 100) for _ in range(3))
    lhs = a.compose(b).compose(c)
    rhs = a.compose(b.compose(c))
    assert (lhs.p - rhs.p).abs().max().item() < 1e-9
    assert (lhs.q - rhs.q).abs().max().item() < 1e-9
    step = random_poses(P, np.random.default_rng(6), 4)
    acc = P.PoseBatch.identity(4)
    for _ in range(10_000):
        acc = acc.compose(step)
    assert (acc.q.norm(dim=1) - 1).abs().max().item() < 1e-9


def test_ref_inverse_cases(P):
    assert P.PoseBatch.identity(3).inverse().allclose(P.PoseBatch.identity(3), atol=0)
    inv = P.PoseBatch.from_pq(position=(1.0, 2.0, 3.0)).inverse()
    assert np.allclose(inv.numpy()[0], [[-1.0, -2.0, -3.0]])
    rng = np.random.default_rng(7)
    p1, p2 = random_poses(P, rng, 10_000), random_poses(P, rng, 10_000)
    got = p1.compose(p2).inverse().compose(p1.inverse()).to_matrix().matrices.cpu().numpy()
    m1, m2 = matrix_oracle(p1), matrix_oracle(p2)
    assert np.abs(got - np.linalg.inv(m1 @ m2) @ np.linalg.inv(m1)).max() < 1e-9


def test_ref_transform_points(P):
    from paper_2410_00425_b200.errors import DimensionError

    pts = np.random.default_rng(8).normal(size=(4, 9, 3))
    assert np.array_equal(P.PoseBatch.identity(4).transform_points(pts).cpu().numpy(), pts)
    half = np.pi / 4
    yaw = P.PoseBatch.from_pq(quaternion=(np.cos(half), 0, 0, np.sin(half)))
    out = yaw.transform_points(np.array([[[1.0, 0.0, 0.0]]])).cpu().numpy()
    assert np.abs(out - np.array([[[0.0, 1.0, 0.0]]])).max() < 1e-12
    rng = np.random.default_rng(9)
    poses = random_poses(P, rng, 200)
    pts = rng.normal(size=(200, 5, 3))
    m = matrix_oracle(poses)
    want = np.einsum("nij,nkj->nki", m[:, :3, :3], pts) + m[:, None, :3, 3]
    assert np.abs(poses.transform_points(pts).cpu().numpy() - want).max() < 1e-9
    with pytest.raises(DimensionError):
        P.PoseBatch.identity(3).transform_points(np.zeros((2, 4, 3)))


def test_ref_matrix_round_trip(P):
    eye = P.PoseBatch.identity(1)
    back = P.PoseBatch.from_matrix(eye.to_matrix().matrices)
    assert torch.equal(back.p, eye.p) and torch.equal(back.q, eye.q)
    for axis in range(3):
        q = np.zeros(4)
        q[axis + 1] = 1.0
        pose = P.PoseBatch.from_pq(quaternion=tuple(q))
        assert P.PoseBatch.from_matrix(pose.to_matrix().matrices).allclose(pose, atol=1e-9)
    poses = random_poses(P, np.random.default_rng(10), 10_000)
    back = P.PoseBatch.from_matrix(poses.to_matrix().matrices)
    assert (back.p - poses.p).abs().max().item() < 1e-9
    assert (back.q - poses.q).abs().max().item() < 1e-9
    bad = np.eye(4)[None].copy()
    bad[0, 0, 0] = 1.1
    with pytest.raises(ValueError, match="orthonormal"):
        P.PoseBatch.from_matrix(bad)
    q = P.quat_normalize(torch.tensor([[-0.5, 0.5, 0.5, 0.5]], dtype=torch.float64).cuda())
    assert q[0, 0] >= 0.0
    q = P.quat_normalize(torch.tensor([[0.0, -1.0, 0.0, 0.0]], dtype=torch.float64).cuda())
    assert q[0, 1] > 0.0


def test_ref_transform_matrix_batch(P):
    bad = np.eye(4)[None].copy()
    bad[0, 3, 0] = 0.5
    with pytest.raises(ValueError, match="bottom row"):
        P.TransformMatrixBatch(bad)
    rng = np.random.default_rng(11)
    a = random_poses(P, rng, 8).to_matrix()
    b = random_poses(P, rng, 8).to_matrix()
    want = a.matrices @ b.matrices
    assert torch.allclose(a.compose(b).matrices, want)
    eye = torch.eye(4, dtype=torch.float64, device=want.device).repeat(8, 1, 1)
    assert torch.allclose(a.inverse().matrices @ a.matrices, eye, atol=1e-12)


# ---- free quaternion functions and TransformMatrixBatch (pose.py:43-164) on the device ----

def test_quaternion_functions_bit_exact(P, pose_golden):
    g = pose_golden
    t = lambda k: torch.tensor(g[k]).cuda()  # noqa: E731
    assert np.array_equal(bits(P.quat_mul(t("qa_norm"), t("qb_norm"))), bits(g["quat_mul"]))
    assert np.array_equal(bits(P.quat_mul(g["qa_raw"], g["qb_raw"])), bits(g["quat_mul_raw"]))
    assert np.array_equal(bits(P.quat_mul(t("qa_norm")[:1], t("qb_norm"))), bits(g["quat_mul_bcast"]))
    nd = P.quat_mul(g["quat_mul_nd_a"], g["quat_mul_nd_b"])
    assert tuple(nd.shape) == (3, 7, 5, 4)
    assert np.array_equal(bits(nd), bits(g["quat_mul_nd"]))
    assert np.array_equal(bits(P.quat_conjugate(g["qa_raw"])), bits(g["quat_conjugate"]))
    assert np.array_equal(bits(P.quat_rotate(t("qa_norm"), t("rot_v"))), bits(g["quat_rotate"]))
    assert np.array_equal(bits(P.quat_rotate(t("qa_norm")[:1], t("rot_v"))), bits(g["quat_rotate_bcast"]))
    assert np.array_equal(bits(P.quat_to_matrix(t("qa_norm"))), bits(g["quat_to_matrix"]))
    assert np.array_equal(bits(P.quat_to_matrix(g["qa_raw"])), bits(g["quat_to_matrix_raw"]))
    assert np.array_equal(bits(P.matrix_to_quat(g["m2q_in"])), bits(g["matrix_to_quat"]))
    from paper_2410_00425_b200.errors import DimensionError

    with pytest.raises(DimensionError):
        P.quat_mul(np.zeros((3, 4)), np.zeros((2, 4)))


def test_transform_matrix_batch_kernels(P, pose_golden):
    g = pose_golden
    A = P.TransformMatrixBatch(g["tm_a"][:1024])
    B = P.TransformMatrixBatch(g["tm_b"][:1024])
    for got, want in ((A.compose(B).matrices, g["tm_compose"][:1024]),
                      (P.TransformMatrixBatch(g["tm_a"][:1]).compose(B).matrices, g["tm_compose_bcast"][:1024]),
                      (A.inverse().matrices, g["tm_inverse"][:1024]),
                      (A.transform_points(g["pts"][:1024]), g["tm_points"][:1024])):
        got = got.cpu().numpy()
        assert np.abs(got - want).max() < 1e-12
    with pytest.raises(ValueError):
        bad = g["tm_a"][:4].copy()
        bad[0, 0, 0] += 1e-3
        P.TransformMatrixBatch(bad)


def test_posebatch_is_immutable(P):
    a = P.PoseBatch(np.zeros((4, 3)), np.tile([1.0, 0, 0, 0], (4, 1)))
    p, q = a.numpy()
    with pytest.raises(ValueError):
        p[0, 0] = 1.0  # read-only host arrays, like the reference (pose.py:195-198)
    a.p[0, 0] = 5.0  # an in-place device write is detected by the next operation
    with pytest.raises(ValueError):
        a.compose(a)
