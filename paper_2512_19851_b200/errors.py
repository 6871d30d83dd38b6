"""Stable error space of the stencil backend.

The numeric codes are the reference's wire codes (pkg/src/elastencil/errors.py:10-164)
so a GPU worker can answer the unchanged coordinator with REPLY_ERR{code} and the
client rebuilds the same typed exception. The same integers are the return values
of the C-ABI (`include/est.h`): 0 = ok, 1 = generic CUDA/NVRTC failure, otherwise
one of the codes below.
"""

from __future__ import annotations


class StencilError(Exception):
    """Base class; code 1 is the generic runtime / CUDA failure."""

    code = 1


def _kind(name: str, code: int, doc: str) -> type:
    cls = type(name, (StencilError,), {"code": code, "__doc__": doc})
    return cls


SelfDependency = _kind("SelfDependency", 10, "statement output is also one of its inputs")
ShapeMismatch = _kind("ShapeMismatch", 11, "slice extents or ranks disagree")
StridedSlice = _kind("StridedSlice", 12, "slice step other than 1")
InvalidSlice = _kind("InvalidSlice", 13, "slice bounds out of range")
InvalidShape = _kind("InvalidShape", 14, "non-positive extent or unsupported rank")
UnsupportedOp = _kind("UnsupportedOp", 15, "operator outside the kernel grammar")
MalformedDag = _kind("MalformedDag", 16, "DAG failed validation")
UnknownArray = _kind("UnknownArray", 17, "array id never created")
IndivisibleShape = _kind("IndivisibleShape", 20, "extent not divisible by the tile count")
OffsetExceedsTileWidth = _kind("OffsetExceedsTileWidth", 21, "ghost depth >= tile width")
StaleMessage = _kind("StaleMessage", 30, "halo for an already-completed round")
PeerLost = _kind("PeerLost", 31, "peer worker vanished outside a rescale")
RescaleUnavailable = _kind("RescaleUnavailable", 40, "worker count cannot be provided")
DaemonUnreachable = _kind("DaemonUnreachable", 41, "memory daemon did not answer")
UnknownAllocation = _kind("UnknownAllocation", 42, "daemon has no such allocation")
RestartFailed = _kind("RestartFailed", 43, "worker set could not be respawned")
SpawnFailed = _kind("SpawnFailed", 50, "a job process failed to start")
PortInUse = _kind("PortInUse", 51, "endpoint already bound")
VersionMismatch = _kind("VersionMismatch", 60, "unsupported frame version")
ProtocolError = _kind("ProtocolError", 61, "frame or body could not be decoded")
SessionFailed = _kind("SessionFailed", 62, "an earlier batch poisoned the session")
OracleMismatch = _kind("OracleMismatch", 70, "result differs from the oracle")

_ALL = [
    StencilError, SelfDependency, ShapeMismatch, StridedSlice, InvalidSlice,
    InvalidShape, UnsupportedOp, MalformedDag, UnknownArray, IndivisibleShape,
    OffsetExceedsTileWidth, StaleMessage, PeerLost, RescaleUnavailable,
    DaemonUnreachable, UnknownAllocation, RestartFailed, SpawnFailed, PortInUse,
    VersionMismatch, ProtocolError, SessionFailed, OracleMismatch,
]
CODES = {cls.code: cls for cls in _ALL}


def from_code(code: int, message: str = "") -> StencilError:
    """Typed exception for a wire / C-ABI code (errors.py:304-307 semantics)."""
    return CODES.get(int(code), StencilError)(message)
