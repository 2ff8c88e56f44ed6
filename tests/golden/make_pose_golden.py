"""Generate tests/golden/pose_golden.npz by running the REFERENCE pose algebra.

Run in the build container (it needs /root/reference, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pose_golden.py

The reference package is loaded read-only through an alias loader (no install, no writes
into /root/reference).  Inputs are seeded; outputs are whatever the reference computes,
so the oracle (oracle/se3.py) and the CUDA kernels are pinned to the reference bits.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

REF_PKG = "/root/reference/pkg/src/batchsim"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pose_golden.npz")


def load_reference():
    sys.dont_write_bytecode = True
    spec = importlib.util.spec_from_file_location(
        "batchsim_ref", os.path.join(REF_PKG, "__init__.py"), submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["batchsim_ref"] = mod
    spec.loader.exec_module(mod)
    import batchsim_ref.pose as pose  # noqa: E402

    return pose


def edge_quats():
    """Degenerate / sign-rule edge cases: zeros in leading slots, -0.0, half turns."""
    qs = [
        [1, 0, 0, 0], [-1, 0, 0, 0], [0, 1, 0, 0], [0, -1, 0, 0], [0, 0, 1, 0], [0, 0, -1, 0],
        [0, 0, 0, 1], [0, 0, 0, -1], [-0.0, -1, 0, 0], [0.0, -0.0, -1, 0], [-0.0, -0.0, -0.0, -2],
        [0, 1, 1, 0], [0, -1, 1, 0], [-0.5, 0.5, 0.5, 0.5], [2, 0, 0, 0], [1e-300, 0, 0, -1e-300],
        [3, -4, 0, 0], [0, 0, -3, 4], [1e150, 1e150, 0, 0], [-1e-150, 2e-150, 0, 0],
    ]
    return np.asarray(qs, dtype=np.float64)


def main():
    pose = load_reference()
    rng = np.random.default_rng(20241017)
    n = 1024
    g = {}
    # random + edge quaternions (raw, unnormalized) and positions
    qa = np.concatenate([rng.normal(size=(n, 4)), edge_quats()])
    qb = np.concatenate([rng.normal(size=(n, 4)), edge_quats()[::-1]])
    pa = rng.uniform(-2, 2, size=qa.shape[:1] + (3,))
    pb = rng.uniform(-2, 2, size=qa.shape[:1] + (3,))
    g["qa_raw"], g["qb_raw"], g["pa"], g["pb"] = qa, qb, pa, pb
    g["qa_norm"] = pose.quat_normalize(qa)
    g["qb_norm"] = pose.quat_normalize(qb)
    A = pose.PoseBatch(pa, qa)
    B = pose.PoseBatch(pb, qb)
    C = A.compose(B)
    g["compose_p"], g["compose_q"] = C.p.copy(), C.q.copy()
    I = A.inverse()
    g["inverse_p"], g["inverse_q"] = I.p.copy(), I.q.copy()
    # the paper's worked expression (P1 P2)^-1 P1^-1
    W = A.compose(B).inverse().compose(A.inverse())
    g["worked_p"], g["worked_q"] = W.p.copy(), W.q.copy()
    # broadcast singleton on each side
    S = pose.PoseBatch(pa[:1], qa[:1])
    g["bcast_left_p"], g["bcast_left_q"] = S.compose(B).p.copy(), S.compose(B).q.copy()
    g["bcast_right_p"], g["bcast_right_q"] = B.compose(S).p.copy(), B.compose(S).q.copy()
    M = A.to_matrix().matrices
    g["to_matrix"] = M.copy()
    F = pose.PoseBatch.from_matrix(M)
    g["from_matrix_p"], g["from_matrix_q"] = F.p.copy(), F.q.copy()
    pts = rng.normal(size=(qa.shape[0], 5, 3))
    g["pts"] = pts
    g["transform_points"] = A.transform_points(pts)
    g["transform_points_single"] = S.transform_points(pts[0])
    # 10^3 chained composes of 4 random steps (norm-drift property, test_pose.py:79-86)
    step = pose.PoseBatch(pa[:4], qa[:4])
    acc = pose.PoseBatch.identity(4)
    for _ in range(1000):
        acc = acc.compose(step)
    g["chain_p"], g["chain_q"] = acc.p.copy(), acc.q.copy()
    # free quaternion functions (pose.py:43-122) and TransformMatrixBatch (pose.py:125-164); a
    # separate stream so the arrays above keep their values
    r2 = np.random.default_rng(7)
    qn_a, qn_b = g["qa_norm"], g["qb_norm"]
    g["quat_mul"] = pose.quat_mul(qn_a, qn_b)
    g["quat_mul_raw"] = pose.quat_mul(qa, qb)                       # unnormalized inputs too
    g["quat_mul_bcast"] = pose.quat_mul(qn_a[:1], qn_b)             # (1,4) x (N,4)
    g["quat_mul_nd_a"] = r2.normal(size=(3, 1, 5, 4))
    g["quat_mul_nd_b"] = r2.normal(size=(1, 7, 5, 4))
    g["quat_mul_nd"] = pose.quat_mul(g["quat_mul_nd_a"], g["quat_mul_nd_b"])  # (3,7,5,4)
    g["quat_conjugate"] = pose.quat_conjugate(qa)
    vs = r2.normal(size=(qa.shape[0], 3))
    g["rot_v"] = vs
    g["quat_rotate"] = pose.quat_rotate(qn_a, vs)
    g["quat_rotate_bcast"] = pose.quat_rotate(qn_a[:1], vs)
    g["quat_to_matrix"] = pose.quat_to_matrix(qn_a)
    g["quat_to_matrix_raw"] = pose.quat_to_matrix(qa)
    # matrix_to_quat on proper rotations, incl. the 180-degree / branch-boundary cases
    rots = np.concatenate([g["quat_to_matrix"], np.stack([np.diag([1.0, -1, -1]), np.diag([-1.0, 1, -1]),
                                                          np.diag([-1.0, -1, 1]), np.eye(3)])])
    g["m2q_in"] = rots
    g["matrix_to_quat"] = pose.matrix_to_quat(rots)
    T = pose.PoseBatch(pa, qa).to_matrix()
    U = pose.PoseBatch(pb, qb).to_matrix()
    g["tm_a"], g["tm_b"] = T.matrices.copy(), U.matrices.copy()
    g["tm_compose"] = T.compose(U).matrices.copy()
    g["tm_compose_bcast"] = pose.TransformMatrixBatch(T.matrices[:1]).compose(U).matrices.copy()
    g["tm_inverse"] = T.inverse().matrices.copy()
    g["tm_points"] = T.transform_points(pts)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
