"""Exception taxonomy of the COVAP API (reference: proj/include/covap/errors.hpp:9-36).

The C-ABI returns one status code per class; ``raise_for_status`` rethrows
the matching Python class so callers keep the reference's error behaviour.
"""


class Error(RuntimeError):
    """Root of all library failures (covap::Error)."""


class InvalidInput(Error):
    """Bad arguments, models, payloads (covap::InvalidInput)."""


class InvalidState(Error):
    """Compressor state does not match the gradient layout (covap::InvalidState)."""


class UndefinedRatio(Error):
    """CCR with zero compute time and nonzero comm (covap::UndefinedRatio)."""


class IncompleteProfile(Error):
    """A distributed profile is missing worker traces (covap::IncompleteProfile)."""


class ConfigError(Error):
    """Configuration problems (covap::ConfigError)."""


class CudaError(Error):
    """CUDA runtime failure inside the native library."""


class NcclError(Error):
    """NCCL failure inside the native library."""


class NoDeviceError(Error):
    """No CUDA device: the B200 path never falls back to the CPU."""


_BY_CODE = {1: InvalidInput, 2: InvalidState, 3: UndefinedRatio, 4: IncompleteProfile,
            5: ConfigError, 6: Error, 10: CudaError, 11: NcclError, 12: NoDeviceError}


def raise_for_status(code, message):
    raise _BY_CODE.get(code, Error)(message)
