"""ctypes binding of the C-ABI library (``include/batchsim_b200.h``).

This is the only module that touches the shared library.  It fails LOUDLY: if the library
is missing or was built for a different ABI, importing the engine's GPU paths raises; there
is no CPU fallback anywhere in the product.  Torch supplies device memory and streams only;
every compute call below passes raw device pointers plus the current torch stream handle.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
# BS_LIB_PATH: an alternative in-tree build of the same library (A/B timing scripts only)
LIB_PATH = os.environ.get("BS_LIB_PATH") or os.path.join(HERE, "_lib", "libbatchsim_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "batchsim_b200.h")
ABI_VERSION = 9

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_F64 = ctypes.c_double
_F32 = ctypes.c_float

# name -> argtypes (restype is always int status, except bs_abi_version).
_SIGNATURES = {
    "bs_abi_version": [],
    "bs_init": [_I32],
    "bs_host_step": [_P, _P, _I64, _I32, _P, _P],
    "bs_quat_normalize_f64": [_P, _I64, _P, _P],
    "bs_quat_normalize_f32": [_P, _I64, _P, _P],
    "bs_pose_compose_f64": [_P, _P, _I64, _P, _P, _I64, _P, _P, _P],
    "bs_pose_compose_f32": [_P, _P, _I64, _P, _P, _I64, _P, _P, _P],
    "bs_pose_inverse_f64": [_P, _P, _I64, _P, _P, _P],
    "bs_pose_inverse_f32": [_P, _P, _I64, _P, _P, _P],
    "bs_pose_transform_points_f64": [_P, _P, _I64, _P, _I64, _I64, _P, _P],
    "bs_pose_transform_points_f32": [_P, _P, _I64, _P, _I64, _I64, _P, _P],
    "bs_pose_to_matrix_f64": [_P, _P, _I64, _P, _P],
    "bs_pose_from_matrix_f64": [_P, _I64, _P, _P, _P, _P],
    "bs_quat_mul_f64": [_P, _I64, _P, _I64, _P, _P],
    "bs_quat_mul_f32": [_P, _I64, _P, _I64, _P, _P],
    "bs_quat_conjugate_f64": [_P, _I64, _P, _P],
    "bs_quat_rotate_f64": [_P, _I64, _P, _I64, _P, _P],
    "bs_quat_rotate_f32": [_P, _I64, _P, _I64, _P, _P],
    "bs_quat_to_matrix_f64": [_P, _I64, _P, _P],
    "bs_matrix_to_quat_f64": [_P, _I64, _P, _P],
    "bs_tmat_compose_f64": [_P, _I64, _P, _I64, _P, _P],
    "bs_tmat_inverse_f64": [_P, _I64, _P, _P],
    "bs_tmat_transform_points_f64": [_P, _I64, _P, _I64, _I64, _P, _P],
}

_lib = None
_initialized_devices: set = set()


def header_symbols() -> list:
    """Every ``bs_*`` function declared in include/batchsim_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int64_t)\s+\**(bs_\w+)\s*\(", text, re.M)))


def register(name: str, argtypes: list) -> None:
    """Add a signature (used by modules that grow the ABI, e.g. sim/render)."""
    _SIGNATURES[name] = argtypes
    if _lib is not None:
        _bind(_lib, name)


def _bind(lib, name):
    fn = getattr(lib, name)
    fn.argtypes = _SIGNATURES[name]
    fn.restype = ctypes.c_int


def load():
    """Load (once) and return the ctypes library handle; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"batchsim-b200 CUDA library not found at {LIB_PATH}; build it with "
            "`python -m paper_2410_00425_b200.build_native` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name in _SIGNATURES:
        _bind(lib, name)
    ver = lib.bs_abi_version()
    if ver != ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI {ver}, expected {ABI_VERSION}; rebuild it")
    _lib = lib
    from . import cabi  # noqa: F401  (registers the struct-taking entry points)
    return lib


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("batchsim-b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch


def ensure_device(device=None) -> int:
    torch = _torch()
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    if idx not in _initialized_devices:
        raise_for_status(load().bs_init(idx), f"bs_init(device={idx})")
        _initialized_devices.add(idx)
    return idx


def stream_handle(device=None) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


def call(name: str, *args) -> None:
    """Invoke a C-ABI entry point and raise the mapped exception on a non-zero status."""
    lib = load()
    status = getattr(lib, name)(*args)
    raise_for_status(status, name)


def ptr(t) -> int:
    """Device pointer of a contiguous CUDA tensor (asserts the contract)."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()
