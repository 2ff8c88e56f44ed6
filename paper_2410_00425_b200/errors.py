"""Engine exception vocabulary.

Mirrors the reference hierarchy (``/root/reference/pkg/src/batchsim/errors.py:4-45``) so
callers that ``except DimensionError`` / ``except ValueError`` keep working after the swap:
every class derives from :class:`BatchSimError` *and* from the builtin the reference pairs it
with.  The C-ABI reports failures as integer status codes (``include/batchsim_b200.h``,
``BS_ERR_*``); :func:`raise_for_status` is the one place those codes become exceptions.
"""

from __future__ import annotations


class BatchSimError(Exception):
    """Root of every error raised by the engine."""


class DimensionError(BatchSimError, ValueError):
    """Batch sizes or trailing dimensions do not line up."""


class AssetParseError(BatchSimError, ValueError):
    """The robot-description text is not well-formed XML (message carries line/column)."""


class SchemaError(BatchSimError, ValueError):
    """Well-formed XML outside the supported URDF/MJCF subset."""


class TopologyError(BatchSimError, ValueError):
    """Links and joints do not form a single tree."""


class SceneBuildError(BatchSimError, ValueError):
    """A per-env scene descriptor cannot be instantiated (message names the env index)."""


class ViewLookupError(BatchSimError, KeyError):
    """A view path did not resolve (message lists the closest names)."""


class LayoutMismatchError(BatchSimError, ValueError):
    """A state snapshot was produced by a different scene layout."""


class DivergenceError(BatchSimError, RuntimeError):
    """Simulation state became non-finite in one or more envs."""


class ModelError(BatchSimError, ValueError):
    """A physical model is invalid (e.g. a dynamic link with no mass)."""


class InputError(BatchSimError, ValueError):
    """Invalid runtime input from the caller (non-finite action, wrong shape)."""


# Status codes shared with include/batchsim_b200.h (BS_OK, BS_ERR_*).
BS_OK = 0
BS_ERR_DIMENSION = 1
BS_ERR_INPUT = 2
BS_ERR_LAYOUT = 3
BS_ERR_CUDA = 4
BS_ERR_ARGUMENT = 5
BS_ERR_UNSUPPORTED = 6

_STATUS_CLASS = {
    BS_ERR_DIMENSION: DimensionError,
    BS_ERR_INPUT: InputError,
    BS_ERR_LAYOUT: LayoutMismatchError,
    BS_ERR_CUDA: RuntimeError,
    BS_ERR_ARGUMENT: ValueError,
    BS_ERR_UNSUPPORTED: ModelError,
}


def raise_for_status(status: int, what: str) -> None:
    """Translate a C-ABI status code into the matching exception (no-op for BS_OK)."""
    if status == BS_OK:
        return
    cls = _STATUS_CLASS.get(status, RuntimeError)
    raise cls(f"{what} failed with status {status}")
