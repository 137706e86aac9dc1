"""Exception types mirroring the reference's (one per spdz_status code).

Reference types: backend.hpp:11-19 (LaneMismatch, TripleShortage,
BackendUnavailable), triple_store.hpp:14-25 (TripleExhausted,
TripleShapeMismatch, MaskExhausted), net.hpp:19-36 (PeerTimeout,
LaneCountMismatch, MalformedShareMessage), spdz.hpp:12-14 (MacCheckFailed),
linear.hpp:10-12 (SliceTooSmall).
"""


class SpdzError(RuntimeError):
    code = -1


class LaneMismatch(SpdzError):
    code = 1


class TripleShortage(SpdzError):
    code = 2


class BackendUnavailable(SpdzError):
    code = 3


class TripleExhausted(SpdzError):
    code = 4


class TripleShapeMismatch(SpdzError):
    code = 5


class MaskExhausted(SpdzError):
    code = 6


class PeerTimeout(SpdzError):
    code = 7


class LaneCountMismatch(SpdzError):
    code = 8


class MalformedShareMessage(SpdzError):
    code = 9


class MacCheckFailed(SpdzError):
    code = 10


class SliceTooSmall(SpdzError):
    code = 11


class StoreFormatError(SpdzError):  # triple_store.hpp:23 (VersionMismatch / CorruptPayload)
    code = 12


class InsufficientTriples(SpdzError):  # preproc.cpp:182-201
    code = 13


class NetError(SpdzError):  # net.hpp:19-30 (NetError, ConnectTimeout, IndexCollision)
    code = 14


class InvalidArgument(SpdzError, ValueError):
    code = 20


class CudaError(SpdzError):
    code = 21


class DealerRejection(SpdzError):
    code = 22


_BY_CODE = {c.code: c for c in (NetError, LaneMismatch, TripleShortage, BackendUnavailable, TripleExhausted,
                                TripleShapeMismatch, MaskExhausted, PeerTimeout, LaneCountMismatch,
                                MalformedShareMessage, MacCheckFailed, SliceTooSmall, StoreFormatError,
                                InsufficientTriples, InvalidArgument, CudaError, DealerRejection)}


def from_code(code: int, msg: str) -> SpdzError:
    cls = _BY_CODE.get(code, SpdzError)
    e = cls(msg)
    e.code = code
    return e
