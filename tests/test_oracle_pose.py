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
