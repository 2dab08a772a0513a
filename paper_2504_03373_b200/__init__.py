"""B200-native GSVD-MUSIC sound-source-localization hot path.

The product is ``_lib/libsslgpu.so`` (CUDA kernels for sm_100a + the C-ABI
engine declared in ``include/sslgpu.h``).  This package holds its build
script and the host-side mirror of the reference's ``ssl::`` API
(``ssl.py``) over that C ABI.
"""
from .errors import DeviceError, IoError, NumericalError, SslError, ValidationError  # noqa: F401

__all__ = ["ssl", "DeviceError", "IoError", "NumericalError", "SslError", "ValidationError"]
