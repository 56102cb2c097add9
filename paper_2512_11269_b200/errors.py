"""Error hierarchy of the operator API, mirroring the reference (errors.py:1-105).

When the reference package `limbforge` is importable, each class here also derives from the
reference class of the same name, so code written against `limbforge.errors` (for example
`except limbforge.errors.LevelMismatch`) catches errors raised by this package unchanged.
"""

try:  # optional: only present where the reference is installed
    from limbforge import errors as _ref
except Exception:  # pragma: no cover - reference absent (e.g. on the GPU box)
    _ref = None


def _base(name, default):
    ref = getattr(_ref, name, None) if _ref is not None else None
    return (ref, default) if ref is not None else (default,)


class LimbforgeError(*_base("LimbforgeError", Exception)):
    """Base class for all errors of the operator API."""


def _mk(name, parent=LimbforgeError, doc=""):
    cls = type(name, _base(name, parent), {"__doc__": doc})
    globals()[name] = cls
    return cls


NoSuchPrimes = _mk("NoSuchPrimes", doc="The prime search under 2^28 ran out of candidates.")
ScaleOverflow = _mk("ScaleOverflow", doc="Encoded coefficients exceed the modulus headroom.")
MissingEvalKey = _mk("MissingEvalKey", doc="A keyswitch needs an evaluation key that was not given.")
LevelMismatch = _mk("LevelMismatch")
ScaleMismatch = _mk("ScaleMismatch")
LevelExhausted = _mk("LevelExhausted")
MissingRotationKey = _mk("MissingRotationKey")
BadStride = _mk("BadStride", doc="Compression stride is not a power of two dividing n.")
NotPeriodic = _mk("NotPeriodic", doc="Slot vector is not exactly periodic with the stride.")
BaseMismatch = _mk("BaseMismatch", doc="Compressed plaintext has no limb for the requested base.")
