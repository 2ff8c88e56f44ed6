"""Oracle pinning: oracle/se3.py reproduces the REFERENCE pose algebra bit for bit.

Golden vectors come from running /root/reference/pkg/src/batchsim/pose.py
(tests/golden/make_pose_golden.py).  CPU only.
"""

import numpy as np
import pytest

from oracle import se3


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def g(pose_golden):
    return pose_golden


def _inputs(g):
    return g["pa"], se3.qnorm(g["qa_raw"]), g["pb"], se3.qnorm(g["qb_raw"])


def test_normalize_bit_exact(g):
    assert np.array_equal(bits(se3.qnorm(g["qa_raw"])), bits(g["qa_norm"]))
    assert np.array_equal(bits(se3.qnorm(g["qb_raw"])), bits(g["qb_norm"]))


def test_compose_inverse_bit_exact(g):
    pa, qa, pb, qb = _inputs(g)
    p, q = se3.compose(pa, qa, pb, qb)
    assert np.array_equal(bits(p), bits(g["compose_p"]))
    assert np.array_equal(bits(q), bits(g["compose_q"]))
    p, q = se3.inverse(pa, qa)
    assert np.array_equal(bits(p), bits(g["inverse_p"]))
    assert np.array_equal(bits(q), bits(g["inverse_q"]))


def test_worked_expression_and_broadcast(g):
    pa, qa, pb, qb = _inputs(g)
    p12, q12 = se3.compose(pa, qa, pb, qb)
    pi, qi = se3.inverse(p12, q12)
    p1i, q1i = se3.inverse(pa, qa)
    p, q = se3.compose(pi, qi, p1i, q1i)
    assert np.array_equal(bits(p), bits(g["worked_p"]))
    assert np.array_equal(bits(q), bits(g["worked_q"]))
    p, q = se3.compose(pa[:1], qa[:1], pb, qb)
    assert np.array_equal(bits(p), bits(g["bcast_left_p"]))
    p, q = se3.compose(pb, qb, pa[:1], qa[:1])
    assert np.array_equal(bits(q), bits(g["bcast_right_q"]))


def test_matrix_round_trip_bit_exact(g):
    pa, qa, _, _ = _inputs(g)
    assert np.array_equal(bits(se3.to_matrix(pa, qa)), bits(g["to_matrix"]))
    p, q = se3.from_matrix(g["to_matrix"])
    assert np.array_equal(bits(p), bits(g["from_matrix_p"]))
    assert np.array_equal(bits(q), bits(g["from_matrix_q"]))


def test_transform_points_tolerance(g):
    # The reference uses einsum (summation order unspecified): the reference's own bound.
    pa, qa, _, _ = _inputs(g)
    got = se3.transform_points(pa, qa, g["pts"])
    want = g["transform_points"]
    fin = np.isfinite(want)
    assert np.array_equal(fin, np.isfinite(got))
    assert np.abs(got[fin] - want[fin]).max() < 1e-12


def test_chain_norm_drift(g):
    pa, qa, _, _ = _inputs(g)
    p = np.zeros((4, 3))
    q = np.tile([1.0, 0, 0, 0], (4, 1))
    for _ in range(1000):
        p, q = se3.compose(p, q, pa[:4], qa[:4])
    assert np.array_equal(bits(p), bits(g["chain_p"]))
    assert np.array_equal(bits(q), bits(g["chain_q"]))


def nanbits(a):
    b = bits(a).copy()
    b[np.isnan(np.asarray(a, np.float64))] = 0x7FF8000000000000
    return b


def test_quaternion_functions_bit_exact(g):
    """pose.py:43-122 free functions: the oracle restatement equals the reference's outputs."""
    assert np.array_equal(nanbits(se3.qmul(g["qa_norm"], g["qb_norm"])), nanbits(g["quat_mul"]))
    assert np.array_equal(nanbits(se3.qmul(g["qa_raw"], g["qb_raw"])), nanbits(g["quat_mul_raw"]))
    assert np.array_equal(nanbits(se3.qmul(g["qa_norm"][:1], g["qb_norm"])), nanbits(g["quat_mul_bcast"]))
    assert np.array_equal(nanbits(se3.qmul(g["quat_mul_nd_a"], g["quat_mul_nd_b"])), nanbits(g["quat_mul_nd"]))
    assert np.array_equal(nanbits(se3.qconj(g["qa_raw"])), nanbits(g["quat_conjugate"]))
    assert np.array_equal(nanbits(se3.qrot(g["qa_norm"], g["rot_v"])), nanbits(g["quat_rotate"]))
    assert np.array_equal(nanbits(se3.qmat(g["qa_norm"])), nanbits(g["quat_to_matrix"]))
    assert np.array_equal(nanbits(se3.qmat(g["qa_raw"])), nanbits(g["quat_to_matrix_raw"]))
    assert np.array_equal(nanbits(se3.mat_to_q(g["m2q_in"])), nanbits(g["matrix_to_quat"]))


def test_transform_matrix_batch_tolerance(g):
    """pose.py:125-164 (matmul / einsum: BLAS summation order is unspecified) to 1e-12."""
    a, b = g["tm_a"], g["tm_b"]
    fin = np.isfinite(g["tm_compose"])
    assert np.abs((a @ b)[fin] - g["tm_compose"][fin]).max() < 1e-12
    r = np.swapaxes(a[:, :3, :3], 1, 2)
    inv = np.tile(np.eye(4), (len(a), 1, 1))
    inv[:, :3, :3] = r
    inv[:, :3, 3] = -np.einsum("nij,nj->ni", r, a[:, :3, 3])
    fin = np.isfinite(g["tm_inverse"])
    assert np.abs(inv[fin] - g["tm_inverse"][fin]).max() < 1e-12
