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


def _dev_tensor(x, last: int, dtype=None) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, np.float64))
    if dtype is not None:
        t = t.to(dtype)
    if t.dtype not in _SUFFIX:
        t = t.to(torch.float64)
    dev = _device(t.device if t.is_cuda else None)
    t = t.to(dev)
    if t.ndim == 0 or t.shape[-1] != last:
        raise DimensionError(f"expected (..., {last}), got {tuple(t.shape)}")
    return t


def _binary(fn, a, la, b, lb, lo):
    """Broadcast (..., la) against (..., lb) like numpy and run the 1-D singleton-broadcast
    kernel `fn` over the flattened batch; returns (..., lo)."""
    try:
        lead = torch.broadcast_shapes(a.shape[:-1], b.shape[:-1])
    except RuntimeError:
        raise DimensionError(f"incompatible batch shapes {tuple(a.shape[:-1])} and {tuple(b.shape[:-1])}") from None

    def flat(x, last):
        if tuple(x.shape[:-1]) == tuple(lead):
            return x.reshape(-1, last).contiguous()
        if x[..., 0].numel() == 1:
            return x.reshape(1, last).contiguous()  # singleton: broadcast inside the kernel
        return x.expand(*lead, last).reshape(-1, last).contiguous()

    fa, fb = flat(a, la), flat(b, lb)
    n = max(fa.shape[0], fb.shape[0]) if fa.shape[0] and fb.shape[0] else 0
    out = torch.empty((n, lo), dtype=a.dtype, device=a.device)
    nat.call(fn, nat.ptr(fa), fa.shape[0], nat.ptr(fb), fb.shape[0], nat.ptr(out), nat.stream_handle())
    return out.reshape(*lead, lo)


def quat_mul(a, b) -> torch.Tensor:
    """pose.py:43-55: Hamilton product of scalar-first quaternions (..., 4), numpy broadcasting,
    on the device (fp64 bit-identical to the reference)."""
    a = _dev_tensor(a, 4)
    b = _dev_tensor(b, 4, a.dtype)
    return _binary(f"bs_quat_mul_{_SUFFIX[a.dtype]}", a, 4, b, 4, 4)


def quat_conjugate(q) -> torch.Tensor:
    """pose.py:58-61 (a new tensor; the input is not modified)."""
    q = _dev_tensor(q, 4, torch.float64)
    flat = q.reshape(-1, 4).contiguous()
    out = torch.empty_like(flat)
    nat.call("bs_quat_conjugate_f64", nat.ptr(flat), flat.shape[0], nat.ptr(out), nat.stream_handle())
    return out.reshape(q.shape)


def quat_rotate(q, v) -> torch.Tensor:
    """pose.py:64-69: rotate vectors (..., 3) by unit quaternions (..., 4), numpy broadcasting."""
    q = _dev_tensor(q, 4)
    v = _dev_tensor(v, 3, q.dtype)
    return _binary(f"bs_quat_rotate_{_SUFFIX[q.dtype]}", q, 4, v, 3, 3)


def quat_to_matrix(q) -> torch.Tensor:
    """pose.py:72-88: rotation matrices (..., 3, 3) from unit quaternions (..., 4)."""
    q = _dev_tensor(q, 4, torch.float64)
    flat = q.reshape(-1, 4).contiguous()
    out = torch.empty((flat.shape[0], 3, 3), dtype=torch.float64, device=q.device)
    nat.call("bs_quat_to_matrix_f64", nat.ptr(flat), flat.shape[0], nat.ptr(out), nat.stream_handle())
    return out.reshape(*q.shape[:-1], 3, 3)


def matrix_to_quat(m) -> torch.Tensor:
    """pose.py:91-122: Shepperd's method (the largest of trace, m00, m11, m22 picks the branch),
    normalized; (..., 3, 3) -> (..., 4)."""
    m = m if isinstance(m, torch.Tensor) else torch.as_tensor(np.asarray(m, np.float64))
    dev = _device(m.device if m.is_cuda else None)
    m = m.to(device=dev, dtype=torch.float64)
    if m.ndim < 2 or tuple(m.shape[-2:]) != (3, 3):
        raise DimensionError(f"expected (..., 3, 3) matrices, got {tuple(m.shape)}")
    flat = m.reshape(-1, 3, 3).contiguous()
    out = torch.empty((flat.shape[0], 4), dtype=torch.float64, device=dev)
    nat.call("bs_matrix_to_quat_f64", nat.ptr(flat), flat.shape[0], nat.ptr(out), nat.stream_handle())
    return out.reshape(*m.shape[:-2], 4)


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
    """N homogeneous 4x4 transforms on the device -- the dense oracle twin (pose.py:125-164).
    compose / inverse / transform_points are bs_tmat_* kernels."""

    def __init__(self, matrices, check: bool = True, device=None):
        dev = _device(device)
        m = matrices if isinstance(matrices, torch.Tensor) else torch.as_tensor(
            np.asarray(matrices, dtype=np.float64))
        m = m.to(device=dev, dtype=torch.float64)
        if m.ndim == 2:
            m = m[None]
        if m.ndim != 3 or tuple(m.shape[1:]) != (4, 4):
            raise DimensionError(f"expected (N, 4, 4) matrices, got {tuple(m.shape)}")
        self.matrices = m.contiguous()
        if check and len(self):
            bottom = self.matrices[:, 3, :]
            want = torch.tensor([0.0, 0.0, 0.0, 1.0], device=dev, dtype=torch.float64)
            if not bool((bottom == want).all()):
                raise ValueError("bottom row must be exactly (0, 0, 0, 1)")
            # R R^T - I from the kernels: (M . M^-1)'s rotation block is R R^T
            rrt = self._compose_raw(self.matrices, self._inverse_raw(self.matrices))[:, :3, :3]
            err = (rrt - torch.eye(3, device=dev, dtype=torch.float64)).abs()
            emax = float(err.max())
            if emax > 1e-8:
                raise ValueError(f"rotation block not orthonormal (max error {emax:.3e})")

    @staticmethod
    def _compose_raw(a, b):
        n = _check_pair(a.shape[0], b.shape[0])
        out = torch.empty((n, 4, 4), dtype=torch.float64, device=a.device)
        nat.call("bs_tmat_compose_f64", nat.ptr(a), a.shape[0], nat.ptr(b), b.shape[0], nat.ptr(out),
                 nat.stream_handle())
        return out

    @staticmethod
    def _inverse_raw(m):
        out = torch.empty_like(m)
        nat.call("bs_tmat_inverse_f64", nat.ptr(m), m.shape[0], nat.ptr(out), nat.stream_handle())
        return out

    def __len__(self) -> int:
        return self.matrices.shape[0]

    def compose(self, other: "TransformMatrixBatch") -> "TransformMatrixBatch":
        return TransformMatrixBatch(self._compose_raw(self.matrices, other.matrices), check=False,
                                    device=self.matrices.device)

    def inverse(self) -> "TransformMatrixBatch":
        return TransformMatrixBatch(self._inverse_raw(self.matrices), check=False, device=self.matrices.device)

    def transform_points(self, pts) -> torch.Tensor:
        pts = torch.as_tensor(pts, dtype=torch.float64, device=self.matrices.device) if not isinstance(
            pts, torch.Tensor) else pts.to(device=self.matrices.device, dtype=torch.float64)
        if pts.ndim == 2:
            pts = pts[None]
        if pts.ndim != 3 or pts.shape[2] != 3:
            raise DimensionError(f"points must have shape (N, K, 3), got {tuple(pts.shape)}")
        pts = pts.contiguous()
        n = _check_pair(len(self), pts.shape[0])
        out = torch.empty((n, pts.shape[1], 3), dtype=torch.float64, device=pts.device)
        nat.call("bs_tmat_transform_points_f64", nat.ptr(self.matrices), len(self), nat.ptr(pts), pts.shape[0],
                 pts.shape[1], nat.ptr(out), nat.stream_handle())
        return out


class PoseBatch:
    """N rigid transforms (position + scalar-first unit quaternion), resident on a GPU.

    Immutable like the reference's read-only arrays (pose.py:195-198): the constructor copies
    its inputs, every operation returns a new batch, and the batch records the version
    counters of its ``p``/``q`` tensors -- an in-place write through them is detected by the
    next operation on the batch, which raises ``ValueError`` instead of computing with the
    modified values.  ``numpy()`` returns read-only arrays, as the reference does.
    """

    __slots__ = ("_p", "_q", "_ver")

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
        self._set(p, q)

    def _set(self, p: torch.Tensor, q: torch.Tensor) -> None:
        self._p, self._q = p, q
        self._ver = (p._version, q._version)

    @classmethod
    def _wrap(cls, p: torch.Tensor, q: torch.Tensor) -> "PoseBatch":
        obj = cls.__new__(cls)
        obj._set(p, q)
        return obj

    @property
    def p(self) -> torch.Tensor:
        """(N, 3) positions (read-only: do not write in place)."""
        return self._p

    @property
    def q(self) -> torch.Tensor:
        """(N, 4) scalar-first unit quaternions (read-only: do not write in place)."""
        return self._q

    def _guard(self) -> "PoseBatch":
        if (self._p._version, self._q._version) != self._ver:
            raise ValueError("PoseBatch is immutable (pose.py:195-198): its p/q tensors were modified in place")
        return self

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
        self._guard()
        other._guard()
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
        self._guard()
        p = torch.empty_like(self.p)
        q = torch.empty_like(self.q)
        if len(self):
            nat.call(f"bs_pose_inverse_{_SUFFIX[self.dtype]}", nat.ptr(self.p), nat.ptr(self.q),
                     len(self), nat.ptr(p), nat.ptr(q), nat.stream_handle())
        return PoseBatch._wrap(p, q)

    def transform_points(self, pts) -> torch.Tensor:
        """R x + t for points (N,K,3) (or (K,3) against a singleton batch)."""
        self._guard()
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
        self._guard()
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
        """(p, q) as read-only float64 numpy arrays (a device->host copy)."""
        self._guard()
        p, q = self.p.double().cpu().numpy(), self.q.double().cpu().numpy()
        p.flags.writeable = False
        q.flags.writeable = False
        return p, q

    def __repr__(self) -> str:
        return f"PoseBatch(n={len(self)}, dtype={self.dtype}, device={self.p.device})"


def stack_poses(poses) -> PoseBatch:
    """Concatenate PoseBatches (pose.py:303-309)."""
    poses = list(poses)
    return PoseBatch._wrap(torch.cat([x.p for x in poses], 0).contiguous(),
                           torch.cat([x.q for x in poses], 0).contiguous())
