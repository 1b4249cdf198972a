"""Typed failures of the B200 region runtime.

The class names and the inheritance tree are the reference's error contract
(`/root/reference/pkg/src/smlrt/errors.py:9-172`): a caller that catches
`smlrt.errors.OutOfBoundsError` catches ours under the same name.  The C-ABI
reports failures as integer status codes (`include/smlrt_b200.h`,
`smlrt_status_t`); `from_status` maps each code back onto one class here so
the Python surface raises exactly what the reference raises.
"""

from __future__ import annotations


class SmlrtError(Exception):
    """Root of every deliberate failure."""


# directive front end (errors.py:15-51)
class DirectiveError(SmlrtError):
    pass


class DirectiveSyntaxError(DirectiveError):
    """Illegal token; `offset` is where the offending token starts."""

    def __init__(self, message, offset, expected=None):
        self.offset = offset
        self.expected = expected
        super().__init__(f"{message} (at offset {offset})")


class SemanticError(DirectiveError):
    pass


class UnboundVariableError(DirectiveError):
    def __init__(self, name, offset=None):
        self.name = name
        self.offset = offset
        super().__init__(f"unbound variable {name!r} in slice bound")


class EmptyRangeError(DirectiveError):
    pass


class UnsupportedConstructError(DirectiveError):
    pass


class MissingClauseError(DirectiveError):
    pass


# data bridge (errors.py:56-79)
class BridgeError(SmlrtError):
    pass


class ArityMismatchError(BridgeError):
    pass


class OutOfBoundsError(BridgeError):
    pass


class FeatureMismatchError(BridgeError):
    pass


class ShapeMismatchError(BridgeError):
    pass


class NonInjectiveScatterError(BridgeError):
    pass


# execution control (errors.py:84-109)
class RuntimeApiError(SmlrtError):
    pass


class DuplicateRegionError(RuntimeApiError):
    pass


class UnknownRegionError(RuntimeApiError):
    pass


class MissingPredicateError(RuntimeApiError):
    pass


class InvalidScheduleError(RuntimeApiError):
    pass


class ModelLoadError(RuntimeApiError):
    pass


class ModelShapeMismatchError(RuntimeApiError):
    pass


# inference engine (errors.py:114-131)
class EngineError(SmlrtError):
    pass


class ManifestError(EngineError):
    pass


class DimChainError(EngineError):
    pass


class NonFiniteWeightsError(EngineError):
    pass


class NonFiniteOutputError(EngineError):
    pass


# record store (errors.py:136-160)
class StoreError(SmlrtError):
    pass


class CorruptManifestError(StoreError):
    pass


class VersionMismatchError(StoreError):
    pass


class ShapeDriftError(StoreError):
    pass


class RangeOutOfBoundsError(StoreError):
    pass


class IoError(SmlrtError):
    pass


class DeviceError(SmlrtError):
    """A CUDA call inside the native library failed (status SMLRT_E_CUDA)."""


# status codes of include/smlrt_b200.h -> exception class
_STATUS = {
    1: ArityMismatchError,
    2: OutOfBoundsError,
    3: FeatureMismatchError,
    4: ShapeMismatchError,
    5: NonInjectiveScatterError,
    6: ModelShapeMismatchError,
    7: NonFiniteOutputError,
    8: DeviceError,
    9: ValueError,
    10: NotImplementedError,
}


def from_status(code: int, message: str) -> Exception:
    cls = _STATUS.get(int(code), SmlrtError)
    return cls(message)
