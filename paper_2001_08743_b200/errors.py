"""Error types mirroring errors.hpp:9-25 (and sampling.cpp:143's std::logic_error)."""


class ConfigError(RuntimeError):
    """Malformed input, schema violation, or inconsistent parameter (errors.hpp:9-12)."""


class BackendError(RuntimeError):
    """A backend / the CUDA device could not be reached or broke its protocol (errors.hpp:15-18)."""


class SpaceExhaustedError(RuntimeError):
    """Every valid configuration has been visited (errors.hpp:22-25)."""


class LogicError(RuntimeError):
    """std::logic_error raised by the reference's Lloyd monotonicity check (sampling.cpp:142-144)."""


class CudaError(BackendError):
    """A CUDA runtime / launch failure inside libktune_cuda."""
