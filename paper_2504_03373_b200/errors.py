"""Error taxonomy of the reference (include/ssl/types.hpp:13-23) plus the
device failure class of the GPU engine.  Exit codes follow the reference CLI
(tools/sslkit.cpp:280-291)."""


class SslError(RuntimeError):
    exit_code = 1


class ValidationError(SslError):
    exit_code = 2


class NumericalError(SslError):
    exit_code = 3


class IoError(SslError):
    exit_code = 4


class DeviceError(SslError):
    """No usable CUDA device / CUDA failure.  There is no CPU fallback."""

    exit_code = 5
