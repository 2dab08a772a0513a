"""ctypes binding of libsslgpu.so (include/sslgpu.h).

The product path: every call lands in the sm_100a engine.  If the library is
missing or no CUDA device is present, calls raise instead of falling back to
any CPU implementation.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DeviceError, IoError, NumericalError, ValidationError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_lib", "libsslgpu.so")

SSLG_OK, SSLG_VALIDATION, SSLG_NUMERICAL, SSLG_IO, SSLG_DEVICE = 0, 2, 3, 4, 5
MAX_M = 64

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


class Config(C.Structure):
    """sslg_config (include/sslgpu.h)."""

    _fields_ = [
        ("m", C.c_uint32),
        ("bins", C.c_uint32),
        ("dirs", C.c_uint32),
        ("window_frames", C.c_uint32),
        ("rebuild_interval", C.c_uint32),
        ("num_sources", C.c_uint32),
        ("denominator_floor", C.c_float),
        ("squared_denominator", C.c_int),
        ("low_power_ratio", C.c_float),
        ("pivoting", C.c_int),
        ("canonical_subspaces", C.c_int),
        ("refine_leading", C.c_int),
        ("precondition", C.c_int),
        ("max_sweeps", C.c_uint32),
        ("max_batch", C.c_uint32),
        ("device", C.c_int),
        ("stream", C.c_void_p),
        ("max_qr_sweeps", C.c_uint32),
        ("tolerance_scale", C.c_float),
        ("compute_residual", C.c_int),
    ]


class StftConfig(C.Structure):
    """sslg_stft_config (include/sslgpu.h; StftConfig, types.hpp:41-52)."""

    _fields_ = [("frame_length", C.c_uint32), ("shift", C.c_uint32), ("window", C.c_int), ("bin_min", C.c_uint32),
                ("bin_max", C.c_uint32)]


class BlockOut(C.Structure):
    _fields_ = [("frame_index", C.c_uint32), ("count", C.c_uint32)]


EXPORTS = {
    "sslg_config_default": (None, [C.POINTER(Config)]),
    "sslg_create": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(Config)]),
    "sslg_destroy": (None, [C.c_void_p]),
    "sslg_last_error": (C.c_char_p, []),
    "sslg_get_config": (C.c_int, [C.c_void_p, C.POINTER(Config)]),
    "sslg_set_noise_model": (C.c_int, [C.c_void_p, _f32p, C.c_int, _u32p]),
    "sslg_set_noise_identity": (C.c_int, [C.c_void_p]),
    "sslg_set_steering": (C.c_int, [C.c_void_p, C.c_uint32, _f32p, _f64p, _u32p, _u32p]),
    "sslg_build_topology": (C.c_int, [_f64p, C.c_uint32, C.c_double, _u32p, _u32p, C.c_uint32, _u32p]),
    "sslg_push_frames": (C.c_int, [C.c_void_p, _f32p, C.c_uint32, C.POINTER(BlockOut), _u32p, _f64p, _u8p, _f64p,
                                   _u32p]),
    "sslg_push_frames_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, _u32p]),
    "sslg_read_results": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(BlockOut), _u32p, _f64p, _u8p, _f64p, _f64p,
                                    _f64p, _u32p, _u8p]),
    "sslg_copy_bin_power_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "sslg_integrate_peaks_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32]),
    "sslg_reset_window": (C.c_int, [C.c_void_p]),
    "sslg_synchronize": (C.c_int, [C.c_void_p]),
    "sslg_correlation": (C.c_int, [C.c_void_p, _f32p, C.c_uint32, _f32p, _u32p]),
    "sslg_gsvd": (C.c_int, [C.c_void_p, _f32p, C.c_uint32, _f64p, _f64p, _u32p, _u8p]),
    "sslg_last_correlation": (C.c_int, [C.c_void_p, _f32p]),
    "sslg_gsvd_ex": (C.c_int, [C.c_void_p, _f32p, C.c_uint32, _f64p, _f64p, _f64p, _u32p, _u8p, _f64p]),
    "sslg_noise_inverse": (C.c_int, [C.c_void_p, C.c_int, _f64p]),
    "sslg_set_async_power": (C.c_int, [C.c_void_p, C.c_int]),
    "sslg_set_spectrum_path": (C.c_int, [C.c_void_p, C.c_int]),
    "sslg_read_correlation_file": (C.c_int, [C.c_char_p, _u32p, _u32p, _u32p, _f32p, C.c_uint64]),
    "sslg_write_correlation_file": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, _f32p]),
    "sslg_load_noise_model": (C.c_int, [C.c_void_p, C.c_char_p, _u32p, _u32p]),
    "sslg_read_steering_file": (C.c_int, [C.c_char_p, _u32p, _u32p, _u32p, _u32p, _f64p, _f32p, C.c_uint64]),
    "sslg_write_steering_file": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _f64p,
                                           _f32p]),
    "sslg_load_steering": (C.c_int, [C.c_void_p, C.c_char_p, _u32p]),
    "sslg_capture_noise_model": (C.c_int, [C.c_void_p, _f32p, C.c_uint64, C.c_int, _f32p, _u32p, _u32p]),
    "sslg_format_estimates_json": (C.c_int, [C.c_uint64, C.c_uint32, _u32p, _f64p, _f64p, _u8p, C.c_char_p,
                                             C.c_uint64, C.POINTER(C.c_uint64)]),
    "sslg_spectrum": (C.c_int, [C.c_void_p, _f64p, C.c_uint32, _f64p, _f64p]),
    "sslg_peaks": (C.c_int, [C.c_void_p, _f64p, C.c_uint32, _u32p, _f64p, _u8p, _u32p]),
    "sslg_last_stage_ms": (C.c_int, [C.c_void_p, _f32p]),
    "sslg_last_launch_count": (C.c_uint32, [C.c_void_p]),
    "sslg_probe_fp64_tflops": (C.c_int, [C.c_int, _f64p]),
    "sslg_probe_fp32_tflops": (C.c_int, [C.c_int, _f64p]),
    "sslg_debug_phase_clocks": (C.c_int, [C.c_void_p, _f64p, C.c_int]),
    "sslg_stft_config_default": (None, [C.POINTER(StftConfig)]),
    "sslg_set_stft": (C.c_int, [C.c_void_p, C.POINTER(StftConfig)]),
    "sslg_stft": (C.c_int, [C.c_void_p, _f32p, C.c_uint64, _f32p, C.c_uint32, _u32p]),
    "sslg_samples_pending": (C.c_int, [C.c_void_p, C.c_uint64, _u32p, _u32p]),
    "sslg_push_samples": (C.c_int, [C.c_void_p, _f32p, C.c_uint64, C.c_uint32, C.POINTER(BlockOut), _u32p, _f64p,
                                    _u8p, _f64p, _u32p]),
    "sslg_locate_samples": (C.c_int, [C.c_void_p, _f32p, C.c_uint64, C.c_uint32, C.POINTER(BlockOut), _u32p,
                                      _f64p, _u8p, _f64p, _u32p]),
    "sslg_push_samples_async": (C.c_int, [C.c_void_p, _f32p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "sslg_wait_results": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(BlockOut), _u32p, _f64p, _u8p,
                                    _f64p, _u32p]),
}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return LIB_PATH


def load(build_if_missing: bool = True) -> C.CDLL:
    """Loads libsslgpu.so (building it in-tree with nvcc if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if not build_if_missing:
                raise DeviceError(f"{LIB_PATH} is missing; run paper_2504_03373_b200/build.py")
            from . import build as _b

            _b.build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


_EXC = {SSLG_VALIDATION: ValidationError, SSLG_NUMERICAL: NumericalError, SSLG_IO: IoError,
        SSLG_DEVICE: DeviceError}


def check(rc: int) -> None:
    if rc == SSLG_OK:
        return
    msg = load().sslg_last_error().decode(errors="replace")
    raise _EXC.get(rc, RuntimeError)(msg)


def ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


f32p = lambda a: ptr(a, _f32p)  # noqa: E731
f64p = lambda a: ptr(a, _f64p)  # noqa: E731
u32p = lambda a: ptr(a, _u32p)  # noqa: E731
u8p = lambda a: ptr(a, _u8p)  # noqa: E731


def c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex64)


def c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)
