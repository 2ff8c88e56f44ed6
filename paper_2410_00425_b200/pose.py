"""Device-resident batched SE(3) poses: the drop-in twin of the reference ``PoseBatch``.

Same surface and semantics as ``/root/reference/pkg/src/batchsim/pose.py``: positions
(N,3) in meters, scalar-first unit quaternions (N,4), renormalised and sign-canonicalised
(first nonzero of w,x,y,z positive) after every operation, singleton broadcasting, and
``DimensionError`` naming both sizes on a mismatch (pose.py:167-174).  The difference is
where the numbers live: ``p``/``q`` are CUDA tensors and every operation is one sm_100a
kernel launch through the C ABI (``bs_pose_*``), asynchronous on the current stream.

Precision: float64 by default (reference parity; normalize/compose/inverse/to_matrix are
bit-identical to numpy); ``dtype=torch.float32`` selects the speed path for
compose/inverse/transform_points.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import DimensionError

_SUFFIX = {torch.float64: "f64", torch.float32: "f32"}


def _device(device):
    nat.ensure_device(device)
    return torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)


def _as_batch(a, last_dim: int, name: str, dtype, device) -> torch.Tensor:
    # pose.py:22-28: 1-D input becomes a batch of one; anything else must be (N, last_dim).
    if isinstance(a, torch.Tensor):
        t = a.detach().to(device=device, dtype=dtype)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float64), device=device).to(dtype)
    if t.ndim == 1:
        t = t[None, :]
    if t.ndim != 2 or t.shape[1] != last_dim:
        raise DimensionError(f"{name} must have shape (N, {last_dim}), got {tuple(t.shape)}")
    return t.contiguous().clone()


def quat_normalize(q) -> torch.Tensor:
    """pose.py:31-40 on the device: q/||q||, then the cascaded sign rule."""
    q = q if isinstance(q, torch.Tensor) else torch.as_tensor(np.asarray(q, np.float64))
    dev = _device(q.device if q.is_cuda else None)
    q = q.to(dev).contiguous()
    flat = q.reshape(-1, 4)
    out = torch.empty_like(flat)
    nat.call(f"bs_quat_normalize_{_SUFFIX[q.dtype]}", nat.ptr(flat), flat.shape[0], nat.ptr(out),
             nat.stream_handle())
    return out.reshape(q.shape)


def quat_conjugate(q: torch.Tensor) -> torch.Tensor:
    out = q.clone()
    out[..., 1:] = -out[..., 1:]
    return out


def _check_pair(na: int, nb: int) -> int:
    # pose.py:167-174: equal sizes, or a singleton side broadcast to the other (incl. 0)
    if na == nb:
        return na
    if na == 1:
        return nb
    if nb == 1:
        return na
    raise DimensionError(f"incompatible batch sizes {na} and {nb}")


class TransformMatrixBatch:
    """N homogeneous 4x4 transforms on the device -- the dense oracle twin (pose.py:125-164)."""

    def __init__(self, matrices, check: bool = True, device=None):
        dev = _device(device)
        m = matrices if isinstance(matrices, torch.Tensor) else torch.as_tensor(
            np.asarray(matrices, dtype=np.float64))
        m = m.to(device=dev, dtype=torch.float64)
        if m.ndim == 2:
            m = m[None]
        if m.ndim != 3 or tuple(m.shape[1:]) != (4, 4):
            raise DimensionError(f"expected (N, 4, 4) matrices, got {tuple(m.shape)}")
        if check:
            bottom = m[:, 3, :]
            want = torch.tensor([0.0, 0.0, 0.0, 1.0], device=dev, dtype=torch.float64)
            if not bool((bottom == want).all()):
                raise ValueError("bottom row must be exactly (0, 0, 0, 1)")
            r = m[:, :3, :3]
            err = (r @ r.transpose(1, 2) - torch.eye(3, device=dev, dtype=torch.float64)).abs()
            emax = float(err.max()) if err.numel() else 0.0
            if emax > 1e-8:
                raise ValueError(f"rotation block not orthonormal (max error {emax:.3e})")
        self.matrices = m.contiguous()

    def __len__(self) -> int:
        return self.matrices.shape[0]

    def compose(self, other: "TransformMatrixBatch") -> "TransformMatrixBatch":
        _check_pair(len(self), len(other))
        return TransformMatrixBatch(torch.matmul(self.matrices, other.matrices), check=False,
                                    device=self.matrices.device)

    def inverse(self) -> "TransformMatrixBatch":
        r = self.matrices[:, :3, :3]
        t = self.matrices[:, :3, 3]
        out = torch.eye(4, dtype=torch.float64, device=r.device).repeat(len(self), 1, 1)
        rt = r.transpose(1, 2)
        out[:, :3, :3] = rt
        out[:, :3, 3] = -(rt @ t[:, :, None])[:, :, 0]
        return TransformMatrixBatch(out, check=False, device=r.device)

    def transform_points(self, pts) -> torch.Tensor:
        pts = torch.as_tensor(pts, dtype=torch.float64, device=self.matrices.device)
        r = self.matrices[:, :3, :3]
        t = self.matrices[:, :3, 3]
        return torch.einsum("nij,nkj->nki", r, pts) + t[:, None, :]


class PoseBatch:
    """N rigid transforms (position + scalar-first unit quaternion), resident on a GPU.

    Immutable by convention: the constructor copies its inputs and every operation returns
    a new batch; the backing tensors are never written after construction.
    """

    __slots__ = ("p", "q")

    def __init__(self, positions, quaternions, _normalize: bool = True, dtype=torch.float64,
                 device=None):
        if isinstance(positions, torch.Tensor) and positions.is_cuda and device is None:
            device = positions.device
        dev = _device(device)
        if dtype not in _SUFFIX:
            raise ValueError(f"unsupported dtype {dtype}")
        p = _as_batch(positions, 3, "positions", dtype, dev)
        q = _as_batch(quaternions, 4, "quaternions", dtype, dev)
        if p.shape[0] != q.shape[0]:
            raise DimensionError(f"positions batch {p.shape[0]} != quaternions batch {q.shape[0]}")
        if _normalize and q.shape[0] > 0:
            nat.call(f"bs_quat_normalize_{_SUFFIX[dtype]}", nat.ptr(q), q.shape[0], nat.ptr(q),
                     nat.stream_handle())
        self.p = p
        self.q = q

    @classmethod
    def _wrap(cls, p: torch.Tensor, q: torch.Tensor) -> "PoseBatch":
        obj = cls.__new__(cls)
        obj.p = p
        obj.q = q
        return obj

    # -- constructors ------------------------------------------------------
    @classmethod
    def identity(cls, n: int = 1, dtype=torch.float64, device=None) -> "PoseBatch":
        dev = _device(device)
        p = torch.zeros((n, 3), dtype=dtype, device=dev)
        q = torch.zeros((n, 4), dtype=dtype, device=dev)
        q[:, 0] = 1.0
        return cls._wrap(p, q)

    @classmethod
    def from_pq(cls, position=(0.0, 0.0, 0.0), quaternion=(1.0, 0.0, 0.0, 0.0),
                dtype=torch.float64, device=None) -> "PoseBatch":
        return cls(np.asarray(position, dtype=np.float64)[None, :],
                   np.asarray(quaternion, dtype=np.float64)[None, :], dtype=dtype, device=device)

    @classmethod
    def from_matrix(cls, matrices, device=None) -> "PoseBatch":
        """pose.py:218-232: (N,4,4) -> poses; rotation block orthonormal within 1e-6."""
        dev = _device(device)
        m = matrices if isinstance(matrices, torch.Tensor) else torch.as_tensor(
            np.asarray(matrices, dtype=np.float64))
        m = m.to(device=dev, dtype=torch.float64)
        if m.ndim == 2:
            m = m[None]
        if m.ndim != 3 or tuple(m.shape[1:]) != (4, 4):
            raise DimensionError(f"expected (N, 4, 4) matrices, got {tuple(m.shape)}")
        m = m.contiguous()
        n = m.shape[0]
        p = torch.empty((n, 3), dtype=torch.float64, device=dev)
        q = torch.empty((n, 4), dtype=torch.float64, device=dev)
        err = torch.zeros((), dtype=torch.float64, device=dev)
        nat.call("bs_pose_from_matrix_f64", nat.ptr(m), n, nat.ptr(p), nat.ptr(q), nat.ptr(err),
                 nat.stream_handle())
        e = float(err)
        if e > 1e-6:
            raise ValueError(f"rotation block not orthonormal within 1e-6 (error {e:.3e})")
        return cls._wrap(p, q)

    # -- core algebra ------------------------------------------------------
    def __len__(self) -> int:
        return self.p.shape[0]

    @property
    def dtype(self):
        return self.p.dtype

    def compose(self, other: "PoseBatch") -> "PoseBatch":
        """self then other in self's frame (== self.to_matrix() @ other.to_matrix())."""
        n = _check_pair(len(self), len(other))
        if other.dtype != self.dtype:
            raise ValueError("compose needs matching dtypes")
        p = torch.empty((n, 3), dtype=self.dtype, device=self.p.device)
        q = torch.empty((n, 4), dtype=self.dtype, device=self.p.device)
        nat.call(f"bs_pose_compose_{_SUFFIX[self.dtype]}", nat.ptr(self.p), nat.ptr(self.q),
                 len(self), nat.ptr(other.p), nat.ptr(other.q), len(other), nat.ptr(p),
                 nat.ptr(q), nat.stream_handle())
        return PoseBatch._wrap(p, q)

    def __mul__(self, other: "PoseBatch") -> "PoseBatch":
        return self.compose(other)

    def inverse(self) -> "PoseBatch":
        p = torch.empty_like(self.p)
        q = torch.empty_like(self.q)
        if len(self):
            nat.call(f"bs_pose_inverse_{_SUFFIX[self.dtype]}", nat.ptr(self.p), nat.ptr(self.q),
                     len(self), nat.ptr(p), nat.ptr(q), nat.stream_handle())
        return PoseBatch._wrap(p, q)

    def transform_points(self, pts) -> torch.Tensor:
        """R x + t for points (N,K,3) (or (K,3) against a singleton batch)."""
        if isinstance(pts, torch.Tensor):
            pts = pts.to(device=self.p.device, dtype=self.dtype)
        else:
            pts = torch.as_tensor(np.asarray(pts, dtype=np.float64), device=self.p.device).to(
                self.dtype)
        if pts.ndim == 2:
            pts = pts[None]
        if pts.ndim != 3 or pts.shape[2] != 3:
            raise DimensionError(f"points must have shape (N, K, 3), got {tuple(pts.shape)}")
        if pts.shape[0] != len(self) and pts.shape[0] != 1 and len(self) != 1:
            raise DimensionError(
                f"points batch {pts.shape[0]} incompatible with pose batch {len(self)}")
        pts = pts.contiguous()
        n = _check_pair(len(self), pts.shape[0])
        out = torch.empty((n, pts.shape[1], 3), dtype=self.dtype, device=self.p.device)
        nat.call(f"bs_pose_transform_points_{_SUFFIX[self.dtype]}", nat.ptr(self.p),
                 nat.ptr(self.q), len(self), nat.ptr(pts), pts.shape[0], pts.shape[1],
                 nat.ptr(out), nat.stream_handle())
        return out

    def to_matrix(self) -> TransformMatrixBatch:
        p, q = self.p.double().contiguous(), self.q.double().contiguous()
        m = torch.empty((len(self), 4, 4), dtype=torch.float64, device=self.p.device)
        if len(self):
            nat.call("bs_pose_to_matrix_f64", nat.ptr(p), nat.ptr(q), len(self), nat.ptr(m),
                     nat.stream_handle())
        return TransformMatrixBatch(m, check=False, device=self.p.device)

    def rotation_matrix(self) -> torch.Tensor:
        return self.to_matrix().matrices[:, :3, :3]

    # -- utilities ---------------------------------------------------------
    def __getitem__(self, idx) -> "PoseBatch":
        p = self.p[idx]
        q = self.q[idx]
        if p.ndim == 1:
            p, q = p[None], q[None]
        return PoseBatch._wrap(p.contiguous(), q.contiguous())

    def allclose(self, other: "PoseBatch", atol: float = 1e-9) -> bool:
        return bool(torch.allclose(self.p, other.p, atol=atol, rtol=1e-5)
                    and torch.allclose(self.q, other.q, atol=atol, rtol=1e-5))

    def numpy(self):
        """(p, q) as float64 numpy arrays (a device->host copy)."""
        return self.p.double().cpu().numpy(), self.q.double().cpu().numpy()

    def __repr__(self) -> str:
        return f"PoseBatch(n={len(self)}, dtype={self.dtype}, device={self.p.device})"


def stack_poses(poses) -> PoseBatch:
    """Concatenate PoseBatches (pose.py:303-309)."""
    poses = list(poses)
    return PoseBatch._wrap(torch.cat([x.p for x in poses], 0).contiguous(),
                           torch.cat([x.q for x in poses], 0).contiguous())
