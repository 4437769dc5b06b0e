"""Exception hierarchy mirroring the reference (REF/errors.py:6-54).

Only the classes the sensing path can raise are mirrored; the C ABI status
codes map onto them in ``_lib.check``.
"""


class TacsimError(Exception):
    """Base class for every error raised by this package (REF/errors.py:6-7)."""


class InvalidArgumentError(TacsimError, ValueError):
    """A caller-supplied argument violates a documented precondition
    (REF/errors.py:10-11).  C ABI status TAC_ERR_INVALID."""


class UnsupportedConfigError(InvalidArgumentError):
    """Valid per the reference but outside what the sm_100a kernels support
    (e.g. a pyramid radius above TAC_MAX_RADIUS).  C ABI TAC_ERR_UNSUPPORTED."""


class CalibrationError(TacsimError):
    """Optical calibration failed to produce a usable table (REF/errors.py:42-43)."""


class NativeLibraryError(TacsimError, RuntimeError):
    """The CUDA library is missing or a CUDA call failed (TAC_ERR_CUDA).

    There is no CPU fallback: the product path fails loudly instead."""
