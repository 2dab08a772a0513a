"""On-disk inputs and output records of the path, through
the C ABI of libsslgpu.so (include/sslgpu.h, csrc/formats.cu):

  SSLC correlation / noise-model tensors  load_correlation, save_correlation
                                          (correlation.cpp:133-193)
  steering-field files                    load_steering, save_steering
                                          (music.cpp:47-106)
  JSONL estimate records                  format_estimates_json
                                          (pipeline.cpp:265-286)

Same names, argument meaning and errors (IoError / ValidationError) as the
reference's functions."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import f32p, f64p, u8p, u32p


def save_correlation(path: str, bins: np.ndarray, t: int) -> None:
    """save_correlation (correlation.cpp:148-167)."""
    bins = np.ascontiguousarray(bins, np.complex64)
    if bins.ndim != 3 or bins.shape[1] != bins.shape[2] or bins.shape[0] == 0:
        from .errors import ValidationError

        raise ValidationError("correlation matrix dimension mismatch")
    _capi.check(_capi.load().sslg_write_correlation_file(path.encode(), bins.shape[1], bins.shape[0], int(t),
                                                         f32p(bins)))


def load_correlation(path: str):
    """load_correlation (correlation.cpp:169-193) -> (CorrelationSet, T)."""
    from .ssl import CorrelationSet

    L = _capi.load()
    m, nb, t = C.c_uint32(), C.c_uint32(), C.c_uint32()
    _capi.check(L.sslg_read_correlation_file(path.encode(), C.byref(m), C.byref(nb), C.byref(t), None, 0))
    arr = np.zeros((nb.value, m.value, m.value), np.complex64)
    _capi.check(L.sslg_read_correlation_file(path.encode(), None, None, None, f32p(arr), arr.size * 2))
    return CorrelationSet(m.value, arr), t.value


def save_steering(path: str, field) -> None:
    """save_steering (music.cpp:47-70): one JSON header line, then float32 pairs."""
    field.validate()
    dirs = np.ascontiguousarray(np.asarray(field.directions, np.float64).reshape(-1, 2))
    vec = np.ascontiguousarray(field.vectors, np.complex64)
    _capi.check(_capi.load().sslg_write_steering_file(path.encode(), field.m, field.bin_min, field.bin_max,
                                                      dirs.shape[0], f64p(dirs), f32p(vec)))


def load_steering(path: str):
    """load_steering (music.cpp:72-106)."""
    from .ssl import SteeringField

    L = _capi.load()
    m, lo, hi, nd = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    _capi.check(L.sslg_read_steering_file(path.encode(), C.byref(m), C.byref(lo), C.byref(hi), C.byref(nd), None,
                                          None, 0))
    dirs = np.zeros((nd.value, 2), np.float64)
    vec = np.zeros((nd.value, hi.value - lo.value + 1, m.value), np.complex64)
    _capi.check(L.sslg_read_steering_file(path.encode(), None, None, None, None, f64p(dirs), f32p(vec), nd.value))
    f = SteeringField(m.value, lo.value, hi.value, dirs, vec)
    f.validate()
    return f


def format_estimates_json(frame_index: int, estimates, directions) -> str:
    """The JSON line run_locate_to_stream writes for one FrameEstimates
    (pipeline.cpp:268-283), as nlohmann::json::dump() lays it out."""
    dirs = np.ascontiguousarray(np.asarray(directions, np.float64).reshape(-1, 2))
    n = len(estimates)
    idx = np.array([e.direction_index for e in estimates], np.uint32)
    pw = np.array([e.power for e in estimates], np.float64)
    low = np.array([1 if e.low_power else 0 for e in estimates], np.uint8)
    L = _capi.load()
    ln = C.c_uint64()
    _capi.check(L.sslg_format_estimates_json(int(frame_index), n, u32p(idx), f64p(dirs), f64p(pw), u8p(low), None, 0,
                                             C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    _capi.check(L.sslg_format_estimates_json(int(frame_index), n, u32p(idx), f64p(dirs), f64p(pw), u8p(low), buf,
                                             ln.value + 1, C.byref(ln)))
    return buf.value.decode()
