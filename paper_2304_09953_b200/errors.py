"""Exception types of the reference API and the C-ABI status mapping.

Names follow proj/include/vscreen/{dock,batcher,chem}.hpp so callers catching
the reference's exceptions keep working.
"""
from __future__ import annotations

from . import _capi


class VscreenError(RuntimeError):
    """Base class (std::runtime_error in the reference)."""


class AtomCountMismatch(VscreenError):
    """dock.hpp:48-51"""


class LengthMismatch(VscreenError):
    """dock.hpp:53-56"""


class EmptyBounds(VscreenError):
    """dock.hpp:58-61"""

    def __init__(self, msg: str = "pocket bounds box is empty"):
        super().__init__(msg)


class OutOfRange(VscreenError):
    """batcher.hpp:42-45"""


class ItemTooLarge(VscreenError):
    """batcher.hpp:47-50"""


class ParseError(VscreenError):
    """chem.hpp:27-37; kind in {UnbalancedBranch, UnclosedRingBond, UnknownToken}."""

    KINDS = ("UnbalancedBranch", "UnclosedRingBond", "UnknownToken")

    def __init__(self, kind: int, position: int, msg: str = ""):
        self.kind = self.KINDS[kind] if 0 <= kind < 3 else "ParseError"
        self.position = position
        super().__init__(f"{self.kind} at position {position}: {msg}".rstrip(": "))


class DisconnectedGraph(VscreenError):
    """chem.hpp:39-42"""


class PocketError(VscreenError):
    """std::runtime_error raised by parse_pocket_json (dock.cpp:414, 441, 448)."""


class CapacityError(VscreenError):
    """A ligand or knob beyond the GPU kernels' limits."""


class DeviceError(VscreenError):
    """CUDA failure or no device."""


class BadFormat(VscreenError):
    """codec::BadFormat (codec.hpp:34-37): a malformed SMZ1 dictionary or
    SMZC library, or a dictionary hash mismatch."""


class UnknownCode(VscreenError):
    """codec::UnknownCode (codec.hpp:23-32): a code byte with no dictionary
    entry; .code and .offset (within the record) as the reference's."""

    def __init__(self, code: int, offset: int):
        super().__init__(f"unknown code byte 0x{code:x} at offset {offset}")
        self.code, self.offset = code, offset


_MAP = {
    _capi.VS_ERR_INVALID_ARGUMENT: ValueError,  # std::invalid_argument
    _capi.VS_ERR_ATOM_COUNT: AtomCountMismatch,
    _capi.VS_ERR_EMPTY_BOUNDS: EmptyBounds,
    _capi.VS_ERR_LENGTH: LengthMismatch,
    _capi.VS_ERR_OUT_OF_RANGE: OutOfRange,
    _capi.VS_ERR_ITEM_TOO_LARGE: ItemTooLarge,
    _capi.VS_ERR_POCKET: PocketError,
    _capi.VS_ERR_CAPACITY: CapacityError,
    _capi.VS_ERR_CUDA: DeviceError,
    _capi.VS_ERR_NO_DEVICE: DeviceError,
    _capi.VS_ERR_STATE: VscreenError,
    _capi.VS_ERR_DISCONNECTED: DisconnectedGraph,
    _capi.VS_ERR_FORMAT: BadFormat,
}


def check(rc: int, handle=None, what: str = "") -> int:
    """Raise the reference-typed exception for a negative status."""
    if rc >= 0:
        return rc
    msg = what
    if handle is not None:
        err = _capi.lib.vs_last_error(handle)
        if err:
            msg = f"{what}: {err.decode()}" if what else err.decode()
    exc = _MAP.get(rc, VscreenError)
    if exc is EmptyBounds:
        raise EmptyBounds()
    raise exc(msg or f"status {rc}")
