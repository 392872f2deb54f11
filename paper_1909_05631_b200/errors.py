"""Exception taxonomy of the reference (sdnnbench/errors.py:8-51), mirrored.

The C ABI returns 2 / 3 / 4 for ParameterError / CapacityError / ShapeError
(include/sdnn.h).  When the reference package is importable the classes
below also derive from its classes, so ``pytest.raises(sdnnbench.errors.
ShapeError)`` in a reference-style test catches ours.
"""

from __future__ import annotations

try:  # optional: only present where the reference is installed
    from sdnnbench import errors as _ref
except Exception:  # noqa: BLE001
    _ref = None


def _bases(name, own):
    ref = getattr(_ref, name, None) if _ref is not None else None
    return (own, ref) if ref is not None and ref is not own else (own,)


# the reference's SdnnError already derives from Exception: listing both
# (Exception, _ref.SdnnError) has no consistent MRO
class SdnnError(*((_ref.SdnnError,) if _ref is not None else (Exception,))):
    """Base class for all package errors."""


class ParameterError(*_bases("ParameterError", SdnnError)):
    """Invalid parameter or parameter combination (CLI exit 2)."""


class CapacityError(*_bases("CapacityError", SdnnError)):
    """Instance exceeds what this code path (or the device) can hold."""


class ShapeError(*_bases("ShapeError", SdnnError)):
    """Dimension mismatch between operands (CLI exit 4)."""


class BoundsError(*_bases("BoundsError", SdnnError)):
    """Index outside the declared matrix extent."""


_BY_CODE = {2: ParameterError, 3: CapacityError, 4: ShapeError}


def from_code(code: int, message: str) -> SdnnError:
    return _BY_CODE.get(code, SdnnError)(message)
