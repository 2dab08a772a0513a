"""On-disk inputs of the path: the SSLC correlation/noise-model tensor
(correlation.cpp:133-193) and the steering-field file (music.cpp:47-106).
Plain host I/O feeding the device engine."""
from __future__ import annotations

import json
import struct

import numpy as np

from .errors import IoError, ValidationError

_MAGIC = b"SSLC"


def save_correlation(path: str, bins: np.ndarray, t: int) -> None:
    """save_correlation (correlation.cpp:148-167): magic, u32 m, bins, T, then
    row-major interleaved float32 per bin."""
    bins = np.ascontiguousarray(bins, np.complex64)
    if bins.ndim != 3 or bins.shape[1] != bins.shape[2] or bins.shape[0] == 0:
        raise ValidationError("correlation matrix dimension mismatch")
    if not np.all(np.isfinite(bins.view(np.float32))):
        raise ValidationError("non-finite correlation entry")
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC)
            f.write(struct.pack("<III", bins.shape[1], bins.shape[0], t))
            f.write(bins.astype("<c8").tobytes())
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e


def load_correlation(path: str):
    """load_correlation (correlation.cpp:169-193) -> (CorrelationSet, T)."""
    from .ssl import CorrelationSet

    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError("cannot open " + path) from e
    if len(data) < 4 or data[:4] != _MAGIC:
        raise IoError(path + ": not a correlation tensor file")
    if len(data) < 16:
        raise IoError(path + ": implausible header")
    m, nb, t = struct.unpack("<III", data[4:16])
    if m < 1 or m > 4096 or nb < 1 or nb > (1 << 20):
        raise IoError(path + ": implausible header")
    need = nb * m * m * 8
    if len(data) - 16 < need:
        raise IoError(path + ": truncated payload")
    arr = np.frombuffer(data[16:16 + need], "<c8").astype(np.complex64).reshape(nb, m, m)
    s = CorrelationSet(m, arr.copy())
    s.validate()
    return s, t


def save_steering(path: str, field) -> None:
    """save_steering (music.cpp:47-70): one JSON header line then float32 pairs."""
    field.validate()
    header = {"bin_max": int(field.bin_max), "bin_min": int(field.bin_min),
              "directions": [[float(a), float(e)] for a, e in np.asarray(field.directions).reshape(-1, 2)],
              "m": int(field.m)}
    try:
        with open(path, "wb") as f:
            f.write(json.dumps(header, separators=(",", ":")).encode() + b"\n")
            f.write(np.ascontiguousarray(field.vectors, np.complex64).astype("<c8").tobytes())
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e


def load_steering(path: str):
    """load_steering (music.cpp:72-106)."""
    from .ssl import SteeringField

    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError("cannot open " + path) from e
    nl = data.find(b"\n")
    if nl < 0:
        raise IoError("missing header line in " + path)
    try:
        h = json.loads(data[:nl])
        m, bmin, bmax = int(h["m"]), int(h["bin_min"]), int(h["bin_max"])
        dirs = np.array([[float(d[0]), float(d[1])] for d in h["directions"]], np.float64).reshape(-1, 2)
    except (ValueError, KeyError, TypeError, IndexError) as e:
        raise IoError(f"bad steering header in {path}: {e}") from e
    if m == 0 or bmax < bmin or len(dirs) == 0:
        raise IoError("bad steering header in " + path)
    count = len(dirs) * (bmax - bmin + 1) * m
    payload = data[nl + 1:]
    if len(payload) < count * 8:
        raise IoError("truncated steering payload in " + path)
    vec = np.frombuffer(payload[: count * 8], "<c8").astype(np.complex64).reshape(len(dirs), bmax - bmin + 1, m)
    f = SteeringField(m, bmin, bmax, dirs, vec.copy())
    f.validate()
    return f
