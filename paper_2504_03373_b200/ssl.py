"""Python mirror of the reference's localization API (namespace ``ssl``,
/root/reference/proj/include/ssl/*.hpp) running on the B200 engine.

Names, argument meanings and error behaviour follow the reference so the
parity tests read like its own tests:

=============================  ==============================================
reference (file:line)          here
=============================  ==============================================
SolverConfig  gsvd.hpp:14-26   :class:`SolverConfig`
NoiseModel    gsvd.hpp:31-50   :class:`NoiseModel` (K^-1 built on the device)
CorrelationSet correlation.hpp:14-21  :class:`CorrelationSet`
CorrelationWindow correlation.hpp:29-51  :class:`CorrelationWindow`
gsvd / gsvd_reference gsvd.hpp:160-163  :func:`gsvd`, :func:`gsvd_reference`
SteeringField music.hpp:32-47  :class:`SteeringField`
MusicConfig   music.hpp:49-62  :class:`MusicConfig`
calc_average_power music.hpp:76-79  :func:`calc_average_power`
DirectionTopology music.hpp:82-86  :class:`DirectionTopology`
peak_search   music.hpp:98-101 :func:`peak_search`
run_locate    pipeline.hpp:71-75  :func:`run_locate` (on STFT frames)
=============================  ==============================================

Every computation goes through libsslgpu.so (``_capi``); nothing here does
numerics on the CPU beyond argument validation and layout bookkeeping.

One deliberate difference: the reference's ``gsvd`` (float Householder + QR)
and ``gsvd_reference`` (double Jacobi) are two solvers; the engine has one,
the FP64 one-sided Jacobi of ``gsvd_reference``.  ``gsvd`` returns its result
narrowed to float (the reference's output type), ``gsvd_reference`` in double.
``SolverConfig.max_qr_sweeps`` / ``tolerance_scale`` configure the QR solver
that the engine does not have; they are validated and otherwise ignored.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import c64, c128, f32p, f64p, u8p, u32p
from .errors import DeviceError, IoError, NumericalError, SslError, ValidationError  # noqa: F401

# ---------------------------------------------------------------------------
# configuration
# ---------------------------------------------------------------------------


@dataclass
class SolverConfig:
    """ssl::SolverConfig (gsvd.hpp:14-26)."""

    max_qr_sweeps: int = 0
    tolerance_scale: float = 1.0
    pivoting: str = "partial"  # partial | none
    compute_residual: bool = False
    canonical_subspaces: bool = True
    # engine-only knob: one A A^H step on the kept span before the canonical
    # complement is built (refine_leading, gsvd.cpp:440-466).  Off by default:
    # the FP64 Jacobi lead vectors are already accurate to FP64 round-off, and
    # the canonical vectors agree with the reference oracle to <= 1e-11 either
    # way (tests/test_gpu_parity.py runs both); on = the generic kernel.
    refine_leading: bool = False
    # engine-only knob: QR-with-column-pivoting preconditioning of the
    # Jacobi (same singular triplets; ~8 instead of ~18 sweeps)
    precondition: bool = True

    def validate(self) -> None:
        if not (self.tolerance_scale > 0):
            raise ValidationError("tolerance_scale must be positive")
        if self.pivoting not in ("partial", "none"):
            raise ValidationError("unknown pivoting mode: " + str(self.pivoting))


@dataclass
class StftConfig:
    """ssl::StftConfig (types.hpp:41-52)."""

    frame_length: int = 512
    shift: int = 160
    window: str = "hann"  # hann | rectangular (stft.cpp:18-26)
    bin_min: int = 16
    bin_max: int = 88

    def bin_count(self) -> int:
        return self.bin_max - self.bin_min + 1

    def validate(self) -> None:
        """StftConfig::validate (stft.cpp:9-16)."""
        if self.frame_length <= 0:
            raise ValidationError("frame_length must be positive")
        if self.shift <= 0:
            raise ValidationError("shift must be positive")
        if self.shift > self.frame_length:
            raise ValidationError("shift must not exceed frame_length")
        if self.bin_min > self.bin_max:
            raise ValidationError("bin_min must not exceed bin_max")
        if self.bin_max > self.frame_length // 2:
            raise ValidationError("bin_max exceeds the half spectrum of frame_length")
        if self.window not in ("hann", "rectangular", "rect"):
            raise ValidationError(f"unknown window '{self.window}'")
        if self.window == "rect":
            self.window = "rectangular"


@dataclass
class MusicConfig:
    """ssl::MusicConfig (music.hpp:49-62)."""

    num_sources: int = 1
    denominator_floor: float = 1e-12
    squared_denominator: bool = False
    low_power_ratio: float = 1.25

    def validate(self) -> None:
        if self.num_sources == 0:
            raise ValidationError("num_sources must be at least 1")
        if not (self.denominator_floor > 0):
            raise ValidationError("denominator_floor must be positive")
        if not (self.low_power_ratio >= 0):
            raise ValidationError("low_power_ratio must be non-negative")


# ---------------------------------------------------------------------------
# containers
# ---------------------------------------------------------------------------


@dataclass
class CorrelationSet:
    """ssl::CorrelationSet: bins [B][m][m] complex64."""

    m: int
    bins: np.ndarray
    frame_index: int = 0

    def bin_count(self) -> int:
        return int(self.bins.shape[0])

    def validate(self) -> None:
        if self.m < 1:
            raise ValidationError("correlation set has no channels")
        if self.bins.shape[0] == 0:
            raise ValidationError("correlation set has no bins")
        if self.bins.shape[1:] != (self.m, self.m):
            raise ValidationError("correlation matrix dimension mismatch")
        if not np.all(np.isfinite(self.bins.view(np.float32))):
            raise ValidationError("non-finite correlation entry")


@dataclass
class Direction:
    azimuth_deg: float = 0.0
    elevation_deg: float = 0.0


@dataclass
class SteeringField:
    """ssl::SteeringField: vectors [dirs][bins][m] complex64."""

    m: int
    bin_min: int
    bin_max: int
    directions: np.ndarray  # [dirs][2] (az, el) degrees
    vectors: np.ndarray

    def bin_count(self) -> int:
        return self.bin_max - self.bin_min + 1

    def validate(self) -> None:
        if self.m == 0:
            raise ValidationError("steering field has no channels")
        if self.bin_max < self.bin_min:
            raise ValidationError("steering field bin range is inverted")
        if len(self.directions) == 0:
            raise ValidationError("steering field has no directions")
        if self.vectors.shape != (len(self.directions), self.bin_count(), self.m):
            raise ValidationError("steering field payload size mismatch")


@dataclass
class GsvdBatch:
    """ssl::GsvdBatch<T> as arrays: singular_values [B][m] (descending),
    e [B][m][m] (column j = left vector j), iterations / converged [B]."""

    singular_values: np.ndarray
    e: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray
    e_r: Optional[np.ndarray] = None  # [B][m][m], row i pairs with value i
    recon_residual: Optional[np.ndarray] = None  # [B]; -1 unless SolverConfig.compute_residual

    @property
    def bins(self) -> int:
        return int(self.singular_values.shape[0])


@dataclass
class MusicSpectrum:
    frame_index: int = 0
    power: np.ndarray = field(default_factory=lambda: np.zeros(0))
    bin_power: Optional[np.ndarray] = None  # [bins][dirs]


@dataclass
class SourceEstimate:
    direction_index: int
    direction: Direction
    power: float
    low_power: bool


@dataclass
class FrameEstimates:
    frame_index: int
    estimates: List[SourceEstimate]


# ---------------------------------------------------------------------------
# device contexts
# ---------------------------------------------------------------------------


class Engine:
    """One device-resident localization stream (an ``sslg_ctx``).

    ``push`` is the hot path: it ingests STFT frames and, for every frame
    that completes the window, runs correlation -> GSVD -> MUSIC ->
    integration -> peak search on the GPU.
    """

    def __init__(self, m: int, bins: int, window_frames: int = 50, music: Optional[MusicConfig] = None,
                 solver: Optional[SolverConfig] = None, max_batch: int = 16, device: int = 0,
                 stream: Optional[int] = None, rebuild_interval: int = 1000):
        self.L = _capi.load()
        music = music or MusicConfig()
        solver = solver or SolverConfig()
        music.validate()
        solver.validate()
        cfg = _capi.Config()
        self.L.sslg_config_default(C.byref(cfg))
        cfg.m, cfg.bins, cfg.window_frames = m, bins, window_frames
        cfg.rebuild_interval = rebuild_interval
        cfg.num_sources = music.num_sources
        cfg.denominator_floor = music.denominator_floor
        cfg.squared_denominator = int(music.squared_denominator)
        cfg.low_power_ratio = music.low_power_ratio
        cfg.pivoting = 1 if solver.pivoting == "partial" else 0
        cfg.canonical_subspaces = int(solver.canonical_subspaces)
        cfg.refine_leading = int(solver.refine_leading)
        cfg.precondition = int(solver.precondition)
        cfg.max_qr_sweeps = int(solver.max_qr_sweeps)
        cfg.tolerance_scale = float(solver.tolerance_scale)
        cfg.compute_residual = int(solver.compute_residual)
        cfg.max_batch = max_batch
        cfg.device = device
        cfg.stream = stream
        h = C.c_void_p()
        _capi.check(self.L.sslg_create(C.byref(h), C.byref(cfg)))
        self.h = h
        self.m, self.bins, self.T = m, bins, window_frames
        self.music = music
        self.max_batch = max_batch
        self.dirs = 0
        self._noise_key = None

    def close(self):
        if getattr(self, "h", None):
            self.L.sslg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # setup ---------------------------------------------------------------
    def set_noise_model(self, k: np.ndarray, check_pd: bool = False) -> None:
        k = c64(k)
        if k.shape != (self.bins, self.m, self.m):
            raise ValidationError("noise model bin count does not match correlation set")
        bad = C.c_uint32(0)
        _capi.check(self.L.sslg_set_noise_model(self.h, f32p(k), int(check_pd), C.byref(bad)))
        self._noise_key = _key(k)

    def set_noise_identity(self) -> None:
        _capi.check(self.L.sslg_set_noise_identity(self.h))
        self._noise_key = ("identity",)

    def set_steering(self, vectors: np.ndarray, directions: Optional[np.ndarray] = None,
                     topology: Optional["DirectionTopology"] = None) -> None:
        vectors = c64(vectors)
        d = vectors.shape[0]
        if vectors.shape[1:] != (self.bins, self.m):
            raise ValidationError("steering field bin count does not match factorization")
        dirs = None if directions is None else np.ascontiguousarray(directions, np.float64)
        off = nbr = None
        if topology is not None:
            off, nbr = topology.offsets, topology.nbr
        elif dirs is None:
            raise ValidationError("directions or a topology are required")
        _capi.check(self.L.sslg_set_steering(self.h, d, f32p(vectors), f64p(dirs), u32p(off),
                                             u32p(nbr if nbr is None or len(nbr) else np.zeros(1, np.uint32))))
        self.dirs = d

    # hot path ----------------------------------------------------------------
    def push(self, frames: np.ndarray, want_power: bool = False):
        """frames [F][m][bins] complex64 on the host; returns a dict of
        per-block estimates (and the broadband power if asked)."""
        frames = c64(frames)
        f = frames.shape[0]
        ns = self.music.num_sources
        n_max = f
        blocks, bptr = _block_buf(n_max)
        idx = np.zeros((n_max, ns), np.uint32)
        pw = np.zeros((n_max, ns))
        low = np.zeros((n_max, ns), np.uint8)
        power = np.zeros((n_max, self.dirs)) if want_power else None
        em = C.c_uint32()
        rc = self.L.sslg_push_frames(self.h, f32p(frames), f, bptr, u32p(idx), f64p(pw), u8p(low), f64p(power),
                                     C.byref(em))
        return _blocks_result(rc, em.value, blocks, idx, pw, low, power)

    # ---- STFT front end (SampleBlock in) -----------------------------------
    def set_stft(self, stft: "StftConfig") -> None:
        """StftConfig (types.hpp:41-52) for push_samples / locate_samples / stft."""
        stft.validate()
        cfg = _capi.StftConfig(stft.frame_length, stft.shift, 0 if stft.window == "hann" else 1, stft.bin_min,
                               stft.bin_max)
        _capi.check(self.L.sslg_set_stft(self.h, C.byref(cfg)))
        self.stft_cfg = stft

    def stft(self, pcm: np.ndarray) -> np.ndarray:
        """stft_stream of one SampleBlock pcm [m][n] float32 -> frames
        [F][m][bins] complex64, bit-identical to the reference (stft.cpp:44-68)."""
        pcm = np.ascontiguousarray(pcm, np.float32)
        n = C.c_uint32()
        _capi.check(self.L.sslg_stft(self.h, f32p(pcm), pcm.shape[1], None, 0, C.byref(n)))
        out = np.zeros((n.value, self.m, self.bins), np.complex64)
        if n.value:
            _capi.check(self.L.sslg_stft(self.h, f32p(pcm), pcm.shape[1], f32p(out), n.value, C.byref(n)))
        return out

    def _samples_call(self, fn, pcm: np.ndarray, want_power: bool):
        pcm = np.ascontiguousarray(pcm, np.float32)
        if pcm.ndim != 2 or pcm.shape[0] != self.m:
            raise ValidationError("sample block channel count does not match the engine")
        nb = C.c_uint32()
        if fn is self.L.sslg_locate_samples:
            fr = C.c_uint32()
            _capi.check(self.L.sslg_stft(self.h, f32p(pcm), pcm.shape[1], None, 0, C.byref(fr)))
            cap = max(fr.value - self.T + 1, 0)
        else:
            _capi.check(self.L.sslg_samples_pending(self.h, pcm.shape[1], None, C.byref(nb)))
            cap = nb.value
        ns = self.music.num_sources
        blocks, bptr = _block_buf(cap)
        idx = np.zeros((cap, ns), np.uint32)
        pw = np.zeros((cap, ns))
        low = np.zeros((cap, ns), np.uint8)
        power = np.zeros((cap, self.dirs)) if want_power else None
        em = C.c_uint32()
        rc = fn(self.h, f32p(pcm), pcm.shape[1], cap, bptr, u32p(idx), f64p(pw), u8p(low), f64p(power),
                C.byref(em))
        return _blocks_result(rc, em.value, blocks, idx, pw, low, power)

    def push_samples(self, pcm: np.ndarray, want_power: bool = False):
        """Streaming: appends pcm [m][n] float32 to the sample history and runs
        every completed frame through the hot path (frames continue across
        calls)."""
        return self._samples_call(self.L.sslg_push_samples, pcm, want_power)

    def locate_samples(self, pcm: np.ndarray, want_power: bool = False):
        """run_locate over one SampleBlock (pipeline.cpp:210-247): fresh window."""
        return self._samples_call(self.L.sslg_locate_samples, pcm, want_power)

    def push_samples_async(self, pcm: np.ndarray) -> int:
        """Enqueues a streaming push without waiting; returns a ticket for
        wait_results.  `pcm` ([m][n] float32) is kept alive until collected
        (pinned memory, e.g. torch .pin_memory().numpy(), overlaps the copy)."""
        pcm = np.ascontiguousarray(pcm, np.float32)
        if pcm.ndim != 2 or pcm.shape[0] != self.m:
            raise ValidationError("sample block channel count does not match the engine")
        t = C.c_uint64()
        _capi.check(self.L.sslg_push_samples_async(self.h, f32p(pcm), pcm.shape[1], C.byref(t)))
        self._inflight = getattr(self, "_inflight", [])
        self._inflight.append((t.value, pcm))
        return t.value

    def set_spectrum_path(self, mode: int = -1) -> None:
        """-1 auto (tcgen05 tf32x3 for grids >= 512 directions), 0 FP64, 1 tcgen05."""
        _capi.check(self.L.sslg_set_spectrum_path(self.h, int(mode)))

    def set_async_power(self, on: bool = True) -> None:
        """Asynchronous pushes also bring the broadband power back (for
        wait_results(want_power=True))."""
        _capi.check(self.L.sslg_set_async_power(self.h, int(on)))

    def wait_results(self, ticket: int, cap: Optional[int] = None, want_power: bool = False):
        """Blocks of every asynchronous push up to `ticket`, in order.  `cap`
        defaults to what the sub-pushes up to `ticket` can emit (max_batch
        blocks each)."""
        ns = self.music.num_sources
        if cap is None:
            cap = max(1, (ticket - getattr(self, "_collected", 0)) * self.max_batch)
        blocks, bptr = _block_buf(cap)
        idx = np.empty((cap, ns), np.uint32)
        pw = np.empty((cap, ns))
        low = np.empty((cap, ns), np.uint8)
        power = np.empty((cap, self.dirs)) if want_power else None
        em = C.c_uint32()
        try:
            _capi.check(self.L.sslg_wait_results(self.h, ticket, cap, bptr, u32p(idx), f64p(pw), u8p(low),
                                                 f64p(power), C.byref(em)))
            self._collected = max(getattr(self, "_collected", 0), ticket)
        finally:
            self._inflight = [(t, a) for t, a in getattr(self, "_inflight", []) if t > ticket]
        n = em.value
        return dict(n=n, frame_index=blocks[:n, 0].copy(), count=blocks[:n, 1].copy(), idx=idx[:n],
                    power_est=pw[:n], low=low[:n].astype(bool), power=None if power is None else power[:n])

    def push_device(self, x_dev_ptr: int, nframes: int) -> int:
        em = C.c_uint32()
        _capi.check(self.L.sslg_push_frames_device(self.h, C.c_void_p(x_dev_ptr), nframes, C.byref(em)))
        return em.value

    def read_results(self, n: int, power=False, bin_power=False, sigma=False):
        ns = self.music.num_sources
        blocks, bptr = _block_buf(n)
        idx = np.zeros((n, ns), np.uint32)
        pw = np.zeros((n, ns))
        low = np.zeros((n, ns), np.uint8)
        P = np.zeros((n, self.dirs)) if power else None
        BP = np.zeros((n, self.bins, self.dirs)) if bin_power else None
        S = np.zeros((n, self.bins, self.m)) if sigma else None
        sw = np.zeros((n, self.bins), np.uint32)
        cv = np.zeros((n, self.bins), np.uint8)
        _capi.check(self.L.sslg_read_results(self.h, n, bptr, u32p(idx), f64p(pw), u8p(low), f64p(P), f64p(BP),
                                             f64p(S), u32p(sw), u8p(cv)))
        return dict(frame_index=blocks[:n, 0].copy(), count=blocks[:n, 1].copy(), idx=idx, power_est=pw,
                    low=low.astype(bool), power=P, bin_power=BP, sigma=S, sweeps=sw, conv=cv.astype(bool))

    def copy_bin_power_device(self, dst_ptr: int, n: int) -> None:
        """Per-bin powers [n][bins][dirs] f64 of the last push -> device buffer."""
        _capi.check(self.L.sslg_copy_bin_power_device(self.h, C.c_void_p(dst_ptr), n))

    def integrate_peaks_device(self, p_ptr: int, n: int, bins_total: int) -> None:
        """Ordered integration + peaks of assembled powers [n][bins_total][dirs] (device)."""
        _capi.check(self.L.sslg_integrate_peaks_device(self.h, C.c_void_p(p_ptr), n, bins_total))

    def reset_window(self):
        _capi.check(self.L.sslg_reset_window(self.h))
        self._inflight = []

    def synchronize(self):
        _capi.check(self.L.sslg_synchronize(self.h))

    def stage_ms(self) -> np.ndarray:
        out = np.zeros(5, np.float32)
        _capi.check(self.L.sslg_last_stage_ms(self.h, f32p(out)))
        return out

    def launch_count(self) -> int:
        return int(self.L.sslg_last_launch_count(self.h))

    # stage entry points --------------------------------------------------------
    def correlation(self, frames: np.ndarray) -> np.ndarray:
        frames = c64(frames)
        f = frames.shape[0]
        out = np.zeros((f, self.bins, self.m, self.m), np.complex64)
        em = C.c_uint32()
        _capi.check(self.L.sslg_correlation(self.h, f32p(frames), f, f32p(out), C.byref(em)))
        return out[: em.value]

    def gsvd(self, r: np.ndarray, want_er: bool = False, want_resid: bool = False):
        """sigma [n][B][m], E [n][B][m][m], sweeps, converged (+ E_r and the
        residual when asked: sslg_gsvd_ex)."""
        r = c64(r)
        if r.ndim == 3:
            r = r[None]
        n = r.shape[0]
        if r.shape[1:] != (self.bins, self.m, self.m):
            raise ValidationError("noise model bin count does not match correlation set")
        sigma = np.zeros((n, self.bins, self.m))
        e = np.zeros((n, self.bins, self.m, self.m), np.complex128)
        er = np.zeros((n, self.bins, self.m, self.m), np.complex128) if want_er else None
        res = np.zeros((n, self.bins)) if want_resid else None
        sw = np.zeros((n, self.bins), np.uint32)
        cv = np.zeros((n, self.bins), np.uint8)
        _capi.check(self.L.sslg_gsvd_ex(self.h, f32p(r), n, f64p(sigma), f64p(e), f64p(er), u32p(sw), u8p(cv),
                                        f64p(res)))
        if want_er or want_resid:
            return sigma, e, sw, cv.astype(bool), er, res
        return sigma, e, sw, cv.astype(bool)

    def load_noise_model(self, path: str) -> int:
        """NoiseModel::from_file (gsvd.cpp:729-734) into this context; returns T."""
        bad, t = C.c_uint32(), C.c_uint32()
        _capi.check(self.L.sslg_load_noise_model(self.h, path.encode(), C.byref(bad), C.byref(t)))
        self._noise_key = ("file", path)
        return t.value

    def load_steering(self, path: str) -> int:
        """load_steering (music.cpp:72-106) into this context; returns bin_min."""
        lo = C.c_uint32()
        _capi.check(self.L.sslg_load_steering(self.h, path.encode(), C.byref(lo)))
        cfg = _capi.Config()
        _capi.check(self.L.sslg_get_config(self.h, C.byref(cfg)))
        self.dirs = cfg.dirs
        return lo.value

    def capture_noise_model(self, pcm: np.ndarray, install: bool = True) -> np.ndarray:
        """capture_noise_model (synth.cpp:329-373) on the device from
        noise-only PCM [m][n]: K [bins][m][m] complex64 (PD-gated); installed
        as this context's noise model unless install=False."""
        pcm = np.ascontiguousarray(pcm, np.float32)
        if pcm.ndim != 2 or pcm.shape[0] != self.m:
            raise ValidationError("sample block channel count does not match the engine")
        k = np.zeros((self.bins, self.m, self.m), np.complex64)
        nf, bad = C.c_uint32(), C.c_uint32()
        _capi.check(self.L.sslg_capture_noise_model(self.h, f32p(pcm), pcm.shape[1], int(install), f32p(k),
                                                    C.byref(nf), C.byref(bad)))
        if install:
            self._noise_key = _key(k)
        return k

    def noise_inverse(self, precision: int = 1) -> np.ndarray:
        """NoiseModel::inverse (0, float) / inverse_double (1): [B][m][m] complex128."""
        out = np.zeros((self.bins, self.m, self.m), np.complex128)
        _capi.check(self.L.sslg_noise_inverse(self.h, int(precision), f64p(out)))
        return out

    def spectrum(self, e: np.ndarray):
        e = c128(e)
        if e.ndim == 3:
            e = e[None]
        n = e.shape[0]
        power = np.zeros((n, self.dirs))
        bp = np.zeros((n, self.bins, self.dirs))
        _capi.check(self.L.sslg_spectrum(self.h, f64p(e), n, f64p(power), f64p(bp)))
        return power, bp

    def peaks(self, power: np.ndarray):
        power = np.ascontiguousarray(power, np.float64)
        if power.ndim == 1:
            power = power[None]
        n = power.shape[0]
        ns = self.music.num_sources
        idx = np.zeros((n, ns), np.uint32)
        pw = np.zeros((n, ns))
        low = np.zeros((n, ns), np.uint8)
        cnt = np.zeros(n, np.uint32)
        _capi.check(self.L.sslg_peaks(self.h, f64p(power), n, u32p(idx), f64p(pw), u8p(low), u32p(cnt)))
        return idx, pw, low.astype(bool), cnt


def _block_buf(n: int):
    """sslg_block_out [n] as a numpy (frame_index, count) array and the
    pointer handed to the C ABI (no per-block ctypes objects)."""
    a = np.zeros((max(n, 1), 2), np.uint32)
    return a, a.ctypes.data_as(C.POINTER(_capi.BlockOut))


def _blocks_result(rc: int, n: int, blocks, idx, pw, low, power):
    """Per-block results of a push.  On an error the blocks emitted before
    it (the frames before the first non-finite one) travel with the
    exception as `.partial`, so run_locate can sink them first like the
    reference's per-frame loop."""
    out = dict(n=n, frame_index=blocks[:n, 0].copy(), count=blocks[:n, 1].copy(), idx=idx[:n], power_est=pw[:n],
               low=low[:n].astype(bool), power=None if power is None else power[:n])
    if rc != _capi.SSLG_OK:
        try:
            _capi.check(rc)
        except Exception as exc:
            exc.partial = out
            raise
    return out


def _key(a: np.ndarray):
    return (a.shape, hash(a.tobytes()))


_ctx_cache: Dict[tuple, Engine] = {}


def _engine(m: int, bins: int, music: Optional[MusicConfig] = None, solver: Optional[SolverConfig] = None,
            max_batch: int = 8, purpose: str = "gsvd") -> Engine:
    """A cached device context per configuration and purpose (the
    peak-search context holds placeholder steering vectors, so it never
    serves a spectrum call)."""
    music = music or MusicConfig()
    solver = solver or SolverConfig()
    key = (purpose, m, bins, music.num_sources, float(music.denominator_floor), bool(music.squared_denominator),
           float(music.low_power_ratio), solver.pivoting, bool(solver.canonical_subspaces),
           bool(solver.refine_leading), bool(solver.precondition), int(solver.max_qr_sweeps),
           float(solver.tolerance_scale), bool(solver.compute_residual), max_batch)
    eng = _ctx_cache.get(key)
    if eng is None:
        eng = Engine(m, bins, window_frames=1, music=music, solver=solver, max_batch=max_batch)
        _ctx_cache[key] = eng
    return eng


# ---------------------------------------------------------------------------
# NoiseModel (gsvd.hpp:31-50, gsvd.cpp:722-780)
# ---------------------------------------------------------------------------


class NoiseModel:
    """ssl::NoiseModel (gsvd.hpp:31-50); the inverses live in device contexts."""

    def __init__(self, k: CorrelationSet):
        self.k = k
        self._prepared: Optional[str] = None

    @staticmethod
    def identity(m: int, bins: int) -> "NoiseModel":
        k = np.zeros((bins, m, m), np.complex64)
        k[:, np.arange(m), np.arange(m)] = 1.0
        return NoiseModel(CorrelationSet(m, k))

    @staticmethod
    def from_file(path: str) -> "NoiseModel":
        from .formats import load_correlation

        n = NoiseModel(load_correlation(path)[0])
        n.check_positive_definite()
        return n

    @staticmethod
    def capture(audio: np.ndarray, stft: "StftConfig") -> "NoiseModel":
        """capture_noise_model (synth.cpp:329-373) from a noise-only
        SampleBlock audio [m][n]: device STFT + FP64 frame sums, bit-identical
        to the reference's K, PD-gated."""
        audio = np.ascontiguousarray(audio, np.float32)
        stft.validate()
        eng = Engine(audio.shape[0], stft.bin_count(), window_frames=1, max_batch=16)
        try:
            eng.set_stft(stft)
            k = eng.capture_noise_model(audio, install=False)
        finally:
            eng.close()
        return NoiseModel(CorrelationSet(audio.shape[0], k))

    def check_positive_definite(self) -> None:
        """Throws NumericalError unless every bin is Hermitian PD (device)."""
        self.k.validate()
        eng = _engine(self.k.m, self.k.bin_count())
        eng.set_noise_model(self.k.bins, check_pd=True)

    def prepare_inverses(self, pivoting: str = "partial") -> None:
        eng = _engine(self.k.m, self.k.bin_count(), solver=SolverConfig(pivoting=pivoting))
        eng.set_noise_model(self.k.bins)
        self._prepared = pivoting


def _bind_noise(eng: Engine, noise: NoiseModel) -> None:
    key = _key(c64(noise.k.bins))
    if eng._noise_key != key:
        eng.set_noise_model(noise.k.bins)


def _check_batch_inputs(noise: NoiseModel, r: CorrelationSet) -> None:
    """check_batch_inputs (gsvd.cpp:799-806)."""
    r.validate()
    noise.k.validate()
    if noise.k.m != r.m:
        raise ValidationError("noise model channel count does not match correlation set")
    if noise.k.bin_count() != r.bin_count():
        raise ValidationError("noise model bin count does not match correlation set")


def gsvd_reference(noise: NoiseModel, r: CorrelationSet, cfg: Optional[SolverConfig] = None,
                   threads: int = 0) -> GsvdBatch:
    """gsvd_reference (gsvd.cpp:832-844) on the device, FP64 results.
    ``threads`` is accepted for signature parity; results never depend on it."""
    cfg = cfg or SolverConfig()
    cfg.validate()
    _check_batch_inputs(noise, r)
    return _gsvd(noise, r, cfg, budget=False)


def _gsvd(noise: NoiseModel, r: CorrelationSet, cfg: SolverConfig, budget: bool) -> GsvdBatch:
    if not budget and cfg.max_qr_sweeps:  # gsvd_reference has no QR budget (gsvd.cpp:832-844)
        cfg = SolverConfig(**{**cfg.__dict__, "max_qr_sweeps": 0})
    eng = _engine(r.m, r.bin_count(), solver=cfg)
    _bind_noise(eng, noise)
    sigma, e, sw, cv, er, res = eng.gsvd(r.bins, want_er=True, want_resid=True)
    return GsvdBatch(sigma[0], e[0], sw[0], cv[0], er[0], res[0])


def gsvd(noise: NoiseModel, r: CorrelationSet, cfg: Optional[SolverConfig] = None, threads: int = 0) -> GsvdBatch:
    """gsvd (gsvd.cpp:810-830): the float-typed batch result; a bin over the
    max_qr_sweeps budget keeps converged = False (gsvd.cpp:819-827)."""
    cfg = cfg or SolverConfig()
    cfg.validate()
    _check_batch_inputs(noise, r)
    b = _gsvd(noise, r, cfg, budget=True)
    return GsvdBatch(b.singular_values.astype(np.float32), b.e.astype(np.complex64), b.iterations, b.converged,
                     b.e_r.astype(np.complex64), b.recon_residual.astype(np.float32))


def calc_average_power(basis: GsvdBatch, steering: SteeringField, cfg: Optional[MusicConfig] = None,
                       keep_bins: bool = False, threads: int = 0) -> MusicSpectrum:
    """calc_average_power (music.cpp:112-165), FP64 on the device."""
    cfg = cfg or MusicConfig()
    cfg.validate()
    steering.validate()
    bins = basis.bins
    if bins != steering.bin_count():
        raise ValidationError("steering field bin count does not match factorization")
    m = steering.m
    if cfg.num_sources >= m:
        raise ValidationError("num_sources must be smaller than the channel count")
    if basis.e.shape[1:] != (m, m):
        raise ValidationError("factorization channel count does not match steering field")
    eng = _engine(m, bins, music=cfg, purpose="spectrum")
    key = ("steer", _key(c64(steering.vectors)))
    if getattr(eng, "_steer_key", None) != key:
        eng.set_steering(steering.vectors, steering.directions)
        eng._steer_key = key
    power, bp = eng.spectrum(basis.e)
    return MusicSpectrum(0, power[0], bp[0] if keep_bins else None)


# ---------------------------------------------------------------------------
# topology + peaks (music.cpp:176-236)
# ---------------------------------------------------------------------------


class DirectionTopology:
    """Neighbor lists as CSR (offsets [D+1], nbr [nnz])."""

    def __init__(self, offsets: np.ndarray, nbr: np.ndarray):
        self.offsets = np.ascontiguousarray(offsets, np.uint32)
        self.nbr = np.ascontiguousarray(nbr, np.uint32)

    @property
    def neighbors(self) -> List[List[int]]:
        return [list(self.nbr[self.offsets[i]:self.offsets[i + 1]]) for i in range(len(self.offsets) - 1)]

    @staticmethod
    def build(directions, radius_deg: float = 10.0) -> "DirectionTopology":
        L = _capi.load()
        dirs = _dirs_array(directions)
        n = dirs.shape[0]
        off = np.zeros(n + 1, np.uint32)
        need = C.c_uint32()
        L.sslg_build_topology(f64p(dirs), n, radius_deg, u32p(off), None, 0, C.byref(need))
        nbr = np.zeros(max(need.value, 1), np.uint32)
        _capi.check(L.sslg_build_topology(f64p(dirs), n, radius_deg, u32p(off), u32p(nbr), need.value,
                                          C.byref(need)))
        return DirectionTopology(off, nbr[: need.value])


def _dirs_array(directions) -> np.ndarray:
    if isinstance(directions, np.ndarray):
        return np.ascontiguousarray(directions, np.float64).reshape(-1, 2)
    return np.array([[d.azimuth_deg, d.elevation_deg] if isinstance(d, Direction) else list(d)
                     for d in directions], np.float64).reshape(-1, 2)


def peak_search(power: np.ndarray, directions, topology: DirectionTopology,
                cfg: Optional[MusicConfig] = None) -> List[SourceEstimate]:
    """peak_search (music.cpp:197-236), on the device."""
    cfg = cfg or MusicConfig()
    cfg.validate()
    power = np.ascontiguousarray(power, np.float64)
    dirs = _dirs_array(directions)
    if power.shape[0] != dirs.shape[0] or len(topology.offsets) - 1 != power.shape[0]:
        raise ValidationError("peak_search input sizes do not match")
    d = power.shape[0]
    eng = _engine(max(cfg.num_sources + 1, 2), 1, music=cfg, purpose="peaks")
    key = ("topo", d, hash(topology.offsets.tobytes()), hash(topology.nbr.tobytes()))
    if getattr(eng, "_topo_key", None) != key:
        dummy = np.zeros((d, 1, eng.m), np.complex64)
        eng.set_steering(dummy, dirs, topology)
        eng._topo_key = key
    idx, pw, low, cnt = eng.peaks(power)
    out = []
    for i in range(int(cnt[0])):
        j = int(idx[0, i])
        out.append(SourceEstimate(j, Direction(*dirs[j]), float(pw[0, i]), bool(low[0, i])))
    return out


# ---------------------------------------------------------------------------
# CorrelationWindow (correlation.cpp:53-130) and run_locate (pipeline.cpp:210-247)
# ---------------------------------------------------------------------------


class CorrelationWindow:
    def __init__(self, t: int, rebuild_interval: int = 1000, m: Optional[int] = None, bins: Optional[int] = None):
        if t < 1:
            raise ValidationError("correlation window length must be >= 1")
        self.t = t
        self.rebuild_interval = max(1, rebuild_interval)
        self._eng: Optional[Engine] = None
        self._pushed = 0
        self._last: Optional[np.ndarray] = None
        self._last_index = 0
        self._shape = None

    def push(self, frame: np.ndarray, frame_index: Optional[int] = None) -> None:
        """frame: SpectrumFrame spectra [m][bins] complex64."""
        frame = c64(frame)
        if frame.ndim != 2 or frame.shape[0] == 0:
            raise ValidationError("empty spectrum frame")
        if self._shape is None:
            self._shape = frame.shape
            self._eng = Engine(frame.shape[0], frame.shape[1], window_frames=self.t,
                               rebuild_interval=self.rebuild_interval, max_batch=1)
        elif frame.shape != self._shape:
            raise ValidationError("spectrum frame shape changed mid-stream")
        r = self._eng.correlation(frame[None])
        self._pushed += 1
        self._last_index = self._pushed - 1 if frame_index is None else frame_index
        if len(r):
            self._last = r[0]

    def filled(self) -> bool:
        return self._pushed >= self.t

    def capacity(self) -> int:
        return self.t

    def normalized(self) -> CorrelationSet:
        if not self.filled():
            raise ValidationError(f"correlation window underfilled: {self._pushed} of {self.t} frames")
        return CorrelationSet(self._shape[0], self._last.copy(), self._last_index)


def run_locate(frames: np.ndarray, window_frames: int, noise: NoiseModel, steering: SteeringField,
               solver: Optional[SolverConfig] = None, music: Optional[MusicConfig] = None,
               sink: Optional[Callable[[FrameEstimates], None]] = None, threads: int = 0,
               topology: Optional[DirectionTopology] = None, max_batch: int = 16,
               first_frame_index: int = 0) -> int:
    """run_locate's streaming loop (pipeline.cpp:210-247) over STFT frames
    [F][m][bins]; returns the number of emitted blocks."""
    music = music or MusicConfig()
    solver = solver or SolverConfig()
    steering.validate()
    if window_frames == 0:
        raise ValidationError("window_frames must be at least 1")
    if noise.k.m != steering.m:
        raise ValidationError("noise model channel count does not match steering field")
    frames = c64(frames)
    if noise.k.bin_count() != frames.shape[2]:
        raise ValidationError("noise model bin count does not match the analysis band")
    eng = Engine(steering.m, steering.bin_count(), window_frames=window_frames, music=music, solver=solver,
                 max_batch=max_batch)
    try:
        eng.set_noise_model(noise.k.bins)
        topo = topology or DirectionTopology.build(steering.directions)
        eng.set_steering(steering.vectors, steering.directions, topo)
        dirs = _dirs_array(steering.directions)
        try:
            out = eng.push(frames)
        except Exception as exc:  # blocks before the failing frame reach the sink first
            _sink_blocks(getattr(exc, "partial", None), dirs, sink, first_frame_index)
            raise
        return _sink_blocks(out, dirs, sink, first_frame_index)
    finally:
        eng.close()


def _sink_blocks(out, dirs, sink, first_frame_index: int = 0) -> int:
    if out is None:
        return 0
    for b in range(out["n"]):
        ests = []
        for i in range(int(out["count"][b])):
            j = int(out["idx"][b, i])
            ests.append(SourceEstimate(j, Direction(*dirs[j]), float(out["power_est"][b, i]), bool(out["low"][b, i])))
        if sink:
            sink(FrameEstimates(first_frame_index + int(out["frame_index"][b]), ests))
    return int(out["n"])


def run_locate_samples(audio: np.ndarray, stft: StftConfig, window_frames: int, noise: NoiseModel,
                       steering: SteeringField, solver: Optional[SolverConfig] = None,
                       music: Optional[MusicConfig] = None, sink: Optional[Callable[[FrameEstimates], None]] = None,
                       threads: int = 0, topology: Optional[DirectionTopology] = None, max_batch: int = 16) -> int:
    """run_locate (pipeline.hpp:71-75, pipeline.cpp:210-247) on a SampleBlock
    audio [m][samples] float32: device STFT -> correlation window -> GSVD ->
    MUSIC -> peaks; the sink receives one FrameEstimates per emitted frame.
    `threads` is accepted for signature parity (results never depend on it)."""
    music = music or MusicConfig()
    solver = solver or SolverConfig()
    steering.validate()
    stft.validate()
    if window_frames == 0:
        raise ValidationError("window_frames must be at least 1")
    if noise.k.m != steering.m:
        raise ValidationError("noise model channel count does not match steering field")
    if noise.k.bin_count() != stft.bin_count():
        raise ValidationError("noise model bin count does not match the analysis band")
    audio = np.ascontiguousarray(audio, np.float32)
    eng = Engine(steering.m, steering.bin_count(), window_frames=window_frames, music=music, solver=solver,
                 max_batch=max_batch)
    try:
        eng.set_noise_model(noise.k.bins)
        topo = topology or DirectionTopology.build(steering.directions)
        eng.set_steering(steering.vectors, steering.directions, topo)
        eng.set_stft(stft)
        dirs = _dirs_array(steering.directions)
        try:
            out = eng.locate_samples(audio)
        except Exception as exc:
            _sink_blocks(getattr(exc, "partial", None), dirs, sink)
            raise
        return _sink_blocks(out, dirs, sink)
    finally:
        eng.close()
