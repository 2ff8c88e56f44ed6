"""batchsim-b200: a B200-native batched simulate-and-render engine.

Drop-in for the data-parallel hot path of ManiSkill3 (arXiv 2410.00425) as the CPU
reference ``batchsim`` specifies it (/root/reference/pkg, /root/reference/SPEC.md):
pose algebra, SoA scene store, fused controller->FK->dynamics->contacts->PGS step,
batched rasterizer with fused pointcloud/segmentation, env sharding.  Compute runs in
hand-written sm_100a CUDA kernels behind the C ABI in include/batchsim_b200.h.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    AssetParseError, BatchSimError, DimensionError, DivergenceError, InputError,
    LayoutMismatchError, ModelError, SceneBuildError, SchemaError, TopologyError,
    ViewLookupError,
)


def __getattr__(name):
    # Lazy: importing the package must not need a GPU; touching the GPU types loads torch
    # and the CUDA library.
    if name in ("PoseBatch", "TransformMatrixBatch", "stack_poses"):
        from . import pose

        return getattr(pose, name)
    raise AttributeError(name)
