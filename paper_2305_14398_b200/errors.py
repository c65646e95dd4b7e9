"""Exception hierarchy mirroring qsim::Error (core/include/qsim/errors.hpp:23-56).

The C ABI returns a qsb_status; :func:`raise_for_status` maps it back onto
these classes, exactly as the C++ adapter maps it onto the qsim:: types.
"""


class Error(RuntimeError):
    """qsim::Error (errors.hpp:23-26)."""


class ShapeError(Error):
    """qsim::ShapeError (errors.hpp:29-32)."""


class ArgumentError(Error):
    """qsim::ArgumentError (errors.hpp:35-38)."""


class LookupError_(Error):
    """qsim::LookupError (errors.hpp:41-44); named with a trailing underscore to
    avoid shadowing the Python builtin."""


class ValidationError(Error):
    """qsim::ValidationError (errors.hpp:47-50)."""


class ResourceError(Error):
    """qsim::ResourceError (errors.hpp:53-56)."""


class DeviceError(Error):
    """A CUDA / NCCL failure below the ABI (qsb_status QSB_ERR_CUDA / QSB_ERR_NCCL)."""


_BY_STATUS = {
    1: ResourceError,
    2: ValidationError,
    3: ShapeError,
    4: ArgumentError,
    5: LookupError_,
    6: DeviceError,
    7: DeviceError,
    8: Error,
}


def raise_for_status(status: int, message: str) -> None:
    if status == 0:
        return
    raise _BY_STATUS.get(status, Error)(message)
