"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the GSVD-MUSIC hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package, and
only as the checker or the timed CPU baseline — never as the thing measured or
shipped.  The product path (``paper_2504_03373_b200``) never imports it.

Two CPU implementations live here:

``port``  — ``sslref.c``: a C restatement of the reference's double-precision
            path (correlation window, Gauss-Jordan inverse, one-sided Jacobi,
            subspace canonicalization, MUSIC spectrum, topology, peaks), each
            function citing /root/reference/proj/src file:line.
``ref``   — ``_ref/libsslref.so``: the UNMODIFIED reference library compiled
            from its own sources by ``oracle/Makefile`` plus ``ref_shim.cpp``
            (a C shim over its public ``ssl::`` API).  Used to pin ``port`` and
            to generate golden fixtures; ships prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsslref.so")
REFERENCE_SRC = "/root/reference/proj"

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the C restatement, and the reference when its sources exist."""
    targets = ["oracle"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _p(a: Optional[np.ndarray], t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# configs mirrored from the reference (include/ssl/gsvd.hpp:14-26,
# include/ssl/music.hpp:49-62)
# ---------------------------------------------------------------------------


class SolverCfg(C.Structure):
    _fields_ = [
        ("max_qr_sweeps", C.c_uint32),
        ("tolerance_scale", C.c_float),
        ("pivoting", C.c_int),
        ("compute_residual", C.c_int),
        ("canonical_subspaces", C.c_int),
    ]

    @classmethod
    def default(cls, **kw):
        s = cls(0, 1.0, 1, 0, 1)
        for k, v in kw.items():
            setattr(s, k, v)
        return s


class MusicCfg(C.Structure):
    _fields_ = [
        ("num_sources", C.c_uint32),
        ("denominator_floor", C.c_float),
        ("squared_denominator", C.c_int),
        ("low_power_ratio", C.c_float),
    ]

    @classmethod
    def make(cls, num_sources=1, floor=1e-12, squared=False, low_power_ratio=1.25):
        return cls(num_sources, floor, int(squared), low_power_ratio)


MAXS = 16


class SceneCfg(C.Structure):
    _fields_ = [
        ("geometry_kind", C.c_int),
        ("mic_count", C.c_uint32),
        ("radius", C.c_double),
        ("frame_length", C.c_uint32),
        ("shift", C.c_uint32),
        ("window", C.c_int),
        ("bin_min", C.c_uint32),
        ("bin_max", C.c_uint32),
        ("sample_rate", C.c_uint32),
        ("duration_s", C.c_double),
        ("seed", C.c_uint64),
        ("has_diffuse", C.c_int),
        ("diffuse_db", C.c_double),
        ("n_sources", C.c_int),
        ("src_az", C.c_double * MAXS),
        ("src_el", C.c_double * MAXS),
        ("src_level_db", C.c_double * MAXS),
        ("src_freq", C.c_double * MAXS),
        ("src_kind", C.c_int * MAXS),
        ("src_noise_role", C.c_int * MAXS),
        ("grid_kind", C.c_int),
        ("grid_step_deg", C.c_double),
        ("sphere_count", C.c_uint32),
        ("el_min_deg", C.c_double),
        ("el_max_deg", C.c_double),
        ("el_step_deg", C.c_double),
        ("noise_kind", C.c_int),
        ("noise_seed", C.c_uint64),
        ("noise_duration_s", C.c_double),
    ]


@dataclass
class Source:
    az: float
    el: float = 0.0
    kind: str = "white"  # tone | white | multitone
    level_db: float = 0.0
    freq: float = 1000.0
    noise_role: bool = False


@dataclass
class Scene:
    """A BASELINE.json-style workload rendered by the reference generators
    (synth.cpp:59-149, 274-373; bench.cpp:178-186)."""

    mics: int = 8
    geometry: str = "circular"  # circular | spherical
    radius: float = 0.05
    frame_length: int = 512
    shift: int = 160
    window: str = "hann"
    bin_min: int = 0
    bin_max: int = 256
    sample_rate: int = 16000
    duration_s: float = 1.0
    seed: int = 7
    diffuse_db: Optional[float] = None
    sources: Sequence[Source] = field(default_factory=list)
    grid: str = "azimuth"  # azimuth | sphere | azel
    grid_step_deg: float = 5.0
    sphere_count: int = 2522
    el_range: tuple = (-90.0, 90.0, 10.0)
    noise: str = "identity"  # identity | captured | random
    noise_seed: int = 0
    noise_duration_s: float = 0.0

    def to_c(self) -> SceneCfg:
        s = SceneCfg()
        s.geometry_kind = 1 if self.geometry == "spherical" else 0
        s.mic_count = self.mics
        s.radius = self.radius
        s.frame_length = self.frame_length
        s.shift = self.shift
        s.window = 0 if self.window == "hann" else 1
        s.bin_min = self.bin_min
        s.bin_max = self.bin_max
        s.sample_rate = self.sample_rate
        s.duration_s = self.duration_s
        s.seed = self.seed
        s.has_diffuse = int(self.diffuse_db is not None)
        s.diffuse_db = self.diffuse_db if self.diffuse_db is not None else -40.0
        s.n_sources = len(self.sources)
        kinds = {"tone": 0, "white": 1, "multitone": 2}
        for i, src in enumerate(self.sources):
            s.src_az[i] = src.az
            s.src_el[i] = src.el
            s.src_level_db[i] = src.level_db
            s.src_freq[i] = src.freq
            s.src_kind[i] = kinds[src.kind]
            s.src_noise_role[i] = int(src.noise_role)
        s.grid_kind = {"azimuth": 0, "sphere": 1, "azel": 2}[self.grid]
        s.grid_step_deg = self.grid_step_deg
        s.sphere_count = self.sphere_count
        s.el_min_deg, s.el_max_deg, s.el_step_deg = self.el_range
        s.noise_kind = {"identity": 0, "captured": 1, "random": 2}[self.noise]
        s.noise_seed = self.noise_seed
        s.noise_duration_s = self.noise_duration_s
        return s


@dataclass
class Workload:
    x: np.ndarray  # [frames][m][bins] complex64 (SpectrumFrame, types.hpp:56-61)
    k: np.ndarray  # [bins][m][m] complex64
    h: np.ndarray  # [dirs][bins][m] complex64
    dirs: np.ndarray  # [dirs][2] float64 (az, el)
    audio: Optional[np.ndarray] = None  # [m][samples] float32

    @property
    def m(self):
        return self.x.shape[1]

    @property
    def bins(self):
        return self.x.shape[2]


# ---------------------------------------------------------------------------
# the compiled reference (oracle/_ref)
# ---------------------------------------------------------------------------


class _Ref:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(path)
        self.L = L
        L.sslref_last_error.restype = C.c_char_p
        L.sslref_workload_new.argtypes = [C.POINTER(SceneCfg), C.POINTER(C.c_void_p)]
        L.sslref_workload_free.argtypes = [C.c_void_p]
        L.sslref_workload_dims.argtypes = [C.c_void_p, _u32p, _u32p, _u32p, _u32p, C.POINTER(C.c_uint64)]
        L.sslref_workload_copy.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, _f64p, _f32p]
        L.sslref_gsvd.argtypes = [_f32p, _f32p, C.c_uint32, C.c_uint32, C.c_int, C.c_uint,
                                  C.POINTER(SolverCfg), _f64p, _f64p, _f64p, _u32p, _u8p, _f64p]
        L.sslref_spectrum.argtypes = [_f64p, C.c_uint32, C.c_uint32, _f32p, C.c_uint32, C.c_int,
                                      C.POINTER(MusicCfg), C.c_uint, _f64p, _f64p]
        L.sslref_locate_frames.argtypes = [_f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _f32p, _f32p,
                                           _f64p, C.c_uint32, C.c_int, C.c_uint, C.POINTER(SolverCfg),
                                           C.POINTER(MusicCfg), _f64p, _f64p, _u32p, _f64p, _u8p, _u32p, _u32p,
                                           _f64p]
        assert L.sslref_sizeof_scene() == C.sizeof(SceneCfg), "SceneCfg layout mismatch"

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.sslref_last_error().decode())

    def workload(self, scene: Scene, with_audio: bool = False) -> Workload:
        h = C.c_void_p()
        sc = scene.to_c()
        self._chk(self.L.sslref_workload_new(C.byref(sc), C.byref(h)))
        try:
            m, b, d, f = (C.c_uint32() for _ in range(4))
            ns = C.c_uint64()
            self.L.sslref_workload_dims(h, C.byref(m), C.byref(b), C.byref(d), C.byref(f), C.byref(ns))
            m, b, d, f = m.value, b.value, d.value, f.value
            x = np.zeros((f, m, b), np.complex64)
            k = np.zeros((b, m, m), np.complex64)
            hv = np.zeros((d, b, m), np.complex64)
            dirs = np.zeros((d, 2), np.float64)
            audio = np.zeros((m, ns.value), np.float32) if with_audio else None
            self.L.sslref_workload_copy(h, _p(x, _f32p), _p(k, _f32p), _p(hv, _f32p), _p(dirs, _f64p),
                                        _p(audio, _f32p))
        finally:
            self.L.sslref_workload_free(h)
        return Workload(x, k, hv, dirs, audio)

    def random_noise_model(self, m, bins, seed) -> np.ndarray:
        k = np.zeros((bins, m, m), np.complex64)
        self._chk(self.L.sslref_random_noise_model(C.c_uint32(m), C.c_uint32(bins), C.c_uint64(seed), _p(k, _f32p)))
        return k

    def random_correlation(self, m, bins, seed) -> np.ndarray:
        r = np.zeros((bins, m, m), np.complex64)
        self._chk(self.L.sslref_random_correlation(C.c_uint32(m), C.c_uint32(bins), C.c_uint64(seed), _p(r, _f32p)))
        return r

    def random_psd_pair(self, m, seed, tag):
        k = np.zeros((m, m), np.complex64)
        r = np.zeros((m, m), np.complex64)
        self.L.sslref_random_psd_pair(C.c_uint32(m), C.c_uint64(seed), C.c_uint64(tag), _p(k, _f32p), _p(r, _f32p))
        return k, r

    def correlation(self, x: np.ndarray, t: int, rebuild_interval: int = 1000) -> np.ndarray:
        x = np.ascontiguousarray(x, np.complex64)
        f, m, b = x.shape
        out = np.zeros((max(f - t + 1, 0), b, m, m), np.complex64)
        n = C.c_uint32()
        self._chk(self.L.sslref_correlation(_p(x, _f32p), C.c_uint32(f), C.c_uint32(m), C.c_uint32(b), C.c_uint32(t),
                                            C.c_uint32(rebuild_interval), _p(out, _f32p), C.byref(n)))
        return out[: n.value]

    def noise_check(self, k: np.ndarray):
        k = np.ascontiguousarray(k, np.complex64)
        self._chk(self.L.sslref_noise_check(_p(k, _f32p), C.c_uint32(k.shape[1]), C.c_uint32(k.shape[0])))

    def mat_inverse(self, k: np.ndarray, precision: int = 1, pivoting: int = 1, bin_label: int = 0):
        k = np.ascontiguousarray(k, np.complex64)
        out = np.zeros(k.shape, np.complex128)
        self._chk(self.L.sslref_mat_inverse(_p(k, _f32p), C.c_uint32(k.shape[0]), C.c_int(precision),
                                            C.c_int(pivoting), C.c_uint32(bin_label), _p(out, _f64p)))
        return out

    def gsvd(self, k, r, path: int = 1, threads: int = 1, solver: Optional[SolverCfg] = None, want_er=False):
        """path 0: ssl::gsvd (float batched), 1: ssl::gsvd_reference (double)."""
        k = np.ascontiguousarray(k, np.complex64)
        r = np.ascontiguousarray(r, np.complex64)
        b, m, _ = r.shape
        sigma = np.zeros((b, m), np.float64)
        e = np.zeros((b, m, m), np.complex128)
        er = np.zeros((b, m, m), np.complex128) if want_er else None
        it = np.zeros(b, np.uint32)
        cv = np.zeros(b, np.uint8)
        res = np.zeros(b, np.float64)
        s = solver or SolverCfg.default()
        self._chk(self.L.sslref_gsvd(_p(k, _f32p), _p(r, _f32p), m, b, path, threads, C.byref(s), _p(sigma, _f64p),
                                     _p(e, _f64p), _p(er, _f64p), _p(it, _u32p), _p(cv, _u8p), _p(res, _f64p)))
        return dict(sigma=sigma, e=e, er=er, iters=it, conv=cv, resid=res)

    def time_gsvd(self, k, r, path: int, threads: int, repeats: int) -> float:
        k = np.ascontiguousarray(k, np.complex64)
        r = np.ascontiguousarray(r, np.complex64)
        b, m, _ = r.shape
        out = C.c_double()
        self._chk(self.L.sslref_time_gsvd(_p(k, _f32p), _p(r, _f32p), C.c_uint32(m), C.c_uint32(b), C.c_int(path),
                                          C.c_uint(threads), C.c_int(repeats), C.byref(out)))
        return out.value

    def save_correlation(self, path: str, k, t: int):
        k = np.ascontiguousarray(k, np.complex64)
        self._chk(self.L.sslref_save_correlation(path.encode(), C.c_uint32(k.shape[1]), C.c_uint32(k.shape[0]),
                                                 C.c_uint32(t), _p(k, _f32p)))

    def load_correlation(self, path: str):
        m, b, t = C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._chk(self.L.sslref_load_correlation(path.encode(), C.byref(m), C.byref(b), C.byref(t), None))
        k = np.zeros((b.value, m.value, m.value), np.complex64)
        self._chk(self.L.sslref_load_correlation(path.encode(), C.byref(m), C.byref(b), C.byref(t), _p(k, _f32p)))
        return k, t.value

    def save_steering(self, path: str, m, bin_min, bin_max, dirs, h):
        dirs = np.ascontiguousarray(dirs, np.float64)
        h = np.ascontiguousarray(h, np.complex64)
        self._chk(self.L.sslref_save_steering(path.encode(), C.c_uint32(m), C.c_uint32(bin_min), C.c_uint32(bin_max),
                                              C.c_uint32(dirs.shape[0]), _p(dirs, _f64p), _p(h, _f32p)))

    def load_steering(self, path: str):
        m, lo, hi, nd = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._chk(self.L.sslref_load_steering(path.encode(), C.byref(m), C.byref(lo), C.byref(hi), C.byref(nd), None,
                                              None))
        dirs = np.zeros((nd.value, 2))
        h = np.zeros((nd.value, hi.value - lo.value + 1, m.value), np.complex64)
        self._chk(self.L.sslref_load_steering(path.encode(), C.byref(m), C.byref(lo), C.byref(hi), C.byref(nd),
                                              _p(dirs, _f64p), _p(h, _f32p)))
        return m.value, lo.value, hi.value, dirs, h

    def format_estimates(self, frame: int, idx, dirs, power, low) -> str:
        idx = np.ascontiguousarray(idx, np.uint32)
        dirs = np.ascontiguousarray(dirs, np.float64)
        power = np.ascontiguousarray(power, np.float64)
        low = np.ascontiguousarray(low, np.uint8)
        buf = C.create_string_buffer(1 << 16)
        self._chk(self.L.sslref_format_estimates(C.c_uint64(frame), C.c_uint32(len(idx)), _p(idx, _u32p),
                                                 _p(dirs, _f64p), _p(power, _f64p), _p(low, _u8p), buf,
                                                 C.c_uint64(1 << 16)))
        return buf.value.decode()

    def time_spectrum(self, k, r, h, music: MusicCfg, threads: int, repeats: int) -> float:
        """Median seconds of calc_average_power<float> on gsvd()'s factors of r."""
        k = np.ascontiguousarray(k, np.complex64)
        r = np.ascontiguousarray(r, np.complex64)
        h = np.ascontiguousarray(h, np.complex64)
        b, m, _ = r.shape
        out = C.c_double()
        self._chk(self.L.sslref_time_spectrum(_p(k, _f32p), _p(r, _f32p), C.c_uint32(m), C.c_uint32(b), _p(h, _f32p),
                                              C.c_uint32(h.shape[0]), C.byref(music), C.c_uint(threads),
                                              C.c_int(repeats), C.byref(out)))
        return out.value

    def gsvd_matrix(self, kinv, r, precision: int, solver: Optional[SolverCfg] = None):
        """precision 0: gsvd_matrix<float>, 1: gsvd_matrix<double>, 2: gsvd_reference_matrix."""
        kinv = np.ascontiguousarray(kinv, np.complex128)
        r = np.ascontiguousarray(r, np.complex128)
        m = r.shape[0]
        sigma = np.zeros(m)
        e = np.zeros((m, m), np.complex128)
        er = np.zeros((m, m), np.complex128)
        it = C.c_uint32()
        cv = C.c_uint8()
        s = solver or SolverCfg.default()
        self._chk(self.L.sslref_gsvd_matrix(_p(kinv, _f64p), _p(r, _f64p), C.c_uint32(m), C.c_int(precision),
                                            C.byref(s), _p(sigma, _f64p), _p(e, _f64p), _p(er, _f64p),
                                            C.byref(it), C.byref(cv)))
        return dict(sigma=sigma, e=e, er=er, iters=it.value, conv=cv.value)

    def jacobi_svd(self, a):
        a = np.ascontiguousarray(a, np.complex128)
        m = a.shape[0]
        sigma = np.zeros(m)
        u = np.zeros((m, m), np.complex128)
        vh = np.zeros((m, m), np.complex128)
        sw = C.c_uint32()
        cv = C.c_uint8()
        self._chk(self.L.sslref_jacobi_svd(_p(a, _f64p), C.c_uint32(m), _p(sigma, _f64p), _p(u, _f64p), _p(vh, _f64p),
                                           C.byref(sw), C.byref(cv)))
        return dict(sigma=sigma, u=u, vh=vh, sweeps=sw.value, conv=cv.value)

    def hermitian_eigenvalues(self, a):
        a = np.ascontiguousarray(a, np.complex128)
        v = np.zeros(a.shape[0])
        self._chk(self.L.sslref_hermitian_eigenvalues(_p(a, _f64p), C.c_uint32(a.shape[0]), _p(v, _f64p)))
        return v

    def spectrum(self, e, h, music: MusicCfg, precision: int = 1, threads: int = 1, keep_bins: bool = False):
        e = np.ascontiguousarray(e, np.complex128)
        h = np.ascontiguousarray(h, np.complex64)
        b, m, _ = e.shape
        d = h.shape[0]
        power = np.zeros(d)
        bp = np.zeros((b, d)) if keep_bins else None
        self._chk(self.L.sslref_spectrum(_p(e, _f64p), m, b, _p(h, _f32p), d, precision, C.byref(music), threads,
                                         _p(power, _f64p), _p(bp, _f64p)))
        return power, bp

    def topology(self, dirs, radius_deg: float = 10.0):
        dirs = np.ascontiguousarray(dirs, np.float64)
        n = dirs.shape[0]
        cap = max(64, n * 64)
        while True:
            off = np.zeros(n + 1, np.uint32)
            nbr = np.zeros(cap, np.uint32)
            rc = self.L.sslref_topology(_p(dirs, _f64p), C.c_uint32(n), C.c_double(radius_deg), _p(off, _u32p),
                                        _p(nbr, _u32p), C.c_uint32(cap))
            if rc == 2 and cap < n * n:
                cap = n * n
                continue
            self._chk(rc)
            return off, nbr[: off[-1]].copy()

    def peaks(self, power, dirs, music: MusicCfg, radius_deg: float = 10.0):
        power = np.ascontiguousarray(power, np.float64)
        dirs = np.ascontiguousarray(dirs, np.float64)
        n = power.shape[0]
        ns = music.num_sources
        idx = np.zeros(ns, np.uint32)
        pw = np.zeros(ns)
        low = np.zeros(ns, np.uint8)
        cnt = C.c_uint32()
        self._chk(self.L.sslref_peaks(_p(power, _f64p), _p(dirs, _f64p), C.c_uint32(n), C.c_double(radius_deg),
                                      C.byref(music), _p(idx, _u32p), _p(pw, _f64p), _p(low, _u8p), C.byref(cnt)))
        c = cnt.value
        return idx[:c].copy(), pw[:c].copy(), low[:c].astype(bool)

    def locate_frames(self, w: Workload, t: int, music: MusicCfg, path: int = 2, threads: int = 1,
                      solver: Optional[SolverCfg] = None, keep_bins: bool = False, max_frames: Optional[int] = None):
        """run_locate's per-frame loop on precomputed frames (pipeline.cpp:227-245).
        path 0 batched float, 1 naive float, 2 reference double."""
        x = np.ascontiguousarray(w.x if max_frames is None else w.x[:max_frames], np.complex64)
        f, m, b = x.shape
        d = w.h.shape[0]
        ne = max(f - t + 1, 0)
        ns = music.num_sources
        power = np.zeros((ne, d))
        bp = np.zeros((ne, b, d)) if keep_bins else None
        idx = np.zeros((ne, ns), np.uint32)
        pw = np.zeros((ne, ns))
        low = np.zeros((ne, ns), np.uint8)
        cnt = np.zeros(ne, np.uint32)
        em = C.c_uint32()
        st = np.zeros(4)
        s = solver or SolverCfg.default()
        k = np.ascontiguousarray(w.k, np.complex64)
        h = np.ascontiguousarray(w.h, np.complex64)
        self._chk(self.L.sslref_locate_frames(_p(x, _f32p), f, m, b, t, _p(k, _f32p), _p(h, _f32p),
                                              _p(np.ascontiguousarray(w.dirs), _f64p), d, path, threads, C.byref(s),
                                              C.byref(music), _p(power, _f64p), _p(bp, _f64p), _p(idx, _u32p),
                                              _p(pw, _f64p), _p(low, _u8p), _p(cnt, _u32p), C.byref(em),
                                              _p(st, _f64p)))
        return dict(power=power, bin_power=bp, idx=idx, pw=pw, low=low.astype(bool), count=cnt, stage_s=st)


# ---------------------------------------------------------------------------
# the C restatement (oracle/_build/liboracle.so)
# ---------------------------------------------------------------------------


class _Port:
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_canonicalize.restype = None

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.orc_last_error().decode())

    def correlation(self, x, t, rebuild_interval=1000):
        x = np.ascontiguousarray(x, np.complex64)
        f, m, b = x.shape
        out = np.zeros((max(f - t + 1, 0), b, m, m), np.complex64)
        n = C.c_uint32()
        self._chk(self.L.orc_correlation(_p(x, _f32p), C.c_uint32(f), C.c_uint32(m), C.c_uint32(b), C.c_uint32(t),
                                         C.c_uint32(rebuild_interval), _p(out, _f32p), C.byref(n)))
        return out[: n.value]

    def stft(self, pcm, frame_length=512, shift=160, window=0, bin_min=16, bin_max=88):
        """stft_stream (stft.cpp:38-68, fft.hpp:15-68): pcm [m][n] -> [F][m][bins] complex64."""
        pcm = np.ascontiguousarray(pcm, np.float32)
        m, n = pcm.shape
        nf = C.c_uint32()
        args = (C.c_uint32(m), C.c_uint64(n), C.c_uint32(frame_length), C.c_uint32(shift), C.c_int(window),
                C.c_uint32(bin_min), C.c_uint32(bin_max))
        self._chk(self.L.orc_stft(_p(pcm, _f32p), *args, None, C.byref(nf)))
        out = np.zeros((nf.value, m, bin_max - bin_min + 1), np.complex64)
        self._chk(self.L.orc_stft(_p(pcm, _f32p), *args, _p(out, _f32p), C.byref(nf)))
        return out

    def mat_inverse(self, k, pivoting=1, bin_label=0):
        k = np.ascontiguousarray(k, np.complex64)
        out = np.zeros(k.shape, np.complex128)
        self._chk(self.L.orc_mat_inverse(_p(k, _f32p), C.c_uint32(k.shape[0]), C.c_int(pivoting),
                                         C.c_uint32(bin_label), _p(out, _f64p)))
        return out

    def jacobi_svd(self, a):
        a = np.ascontiguousarray(a, np.complex128)
        m = a.shape[0]
        sigma = np.zeros(m)
        u = np.zeros((m, m), np.complex128)
        vh = np.zeros((m, m), np.complex128)
        sw = C.c_uint32()
        cv = C.c_uint8()
        self._chk(self.L.orc_jacobi_svd(_p(a, _f64p), C.c_uint32(m), _p(sigma, _f64p), _p(u, _f64p), _p(vh, _f64p),
                                        C.byref(sw), C.byref(cv)))
        return dict(sigma=sigma, u=u, vh=vh, sweeps=sw.value, conv=cv.value)

    def gsvd_reference(self, k, r, canonical=True, threads=None, kinv=None, want_er=False):
        k = np.ascontiguousarray(k, np.complex64)
        r = np.ascontiguousarray(r, np.complex64)
        b, m, _ = r.shape
        sigma = np.zeros((b, m))
        e = np.zeros((b, m, m), np.complex128)
        er = np.zeros((b, m, m), np.complex128) if want_er else None
        sw = np.zeros(b, np.uint32)
        cv = np.zeros(b, np.uint8)
        kinv_p = None
        if kinv is not None:
            kinv = np.ascontiguousarray(kinv, np.complex128)
            kinv_p = _p(kinv, _f64p)
        th = threads or os.cpu_count() or 1
        self._chk(self.L.orc_gsvd_reference(_p(k, _f32p), kinv_p, _p(r, _f32p), C.c_uint32(m), C.c_uint32(b),
                                            C.c_int(int(canonical)), C.c_int(th), _p(sigma, _f64p), _p(e, _f64p),
                                            _p(er, _f64p), _p(sw, _u32p), _p(cv, _u8p)))
        return dict(sigma=sigma, e=e, er=er, sweeps=sw, conv=cv)

    def spectrum(self, e, h, num_sources, floor=1e-12, squared=False, threads=None, keep_bins=False):
        e = np.ascontiguousarray(e, np.complex128)
        h = np.ascontiguousarray(h, np.complex64)
        b, m, _ = e.shape
        d = h.shape[0]
        power = np.zeros(d)
        bp = np.zeros((b, d)) if keep_bins else None
        th = threads or os.cpu_count() or 1
        self._chk(self.L.orc_spectrum(_p(e, _f64p), C.c_uint32(m), C.c_uint32(b), _p(h, _f32p), C.c_uint32(d),
                                      C.c_uint32(num_sources), C.c_float(floor), C.c_int(int(squared)), C.c_int(th),
                                      _p(power, _f64p), _p(bp, _f64p)))
        return power, bp

    def topology(self, dirs, radius_deg=10.0):
        dirs = np.ascontiguousarray(dirs, np.float64)
        n = dirs.shape[0]
        cap = n * n + 1
        off = np.zeros(n + 1, np.uint32)
        nbr = np.zeros(cap, np.uint32)
        self._chk(self.L.orc_topology(_p(dirs, _f64p), C.c_uint32(n), C.c_double(radius_deg), _p(off, _u32p),
                                      _p(nbr, _u32p), C.c_uint32(cap)))
        return off, nbr[: off[-1]].copy()

    def peaks(self, power, offsets, nbr, num_sources, low_power_ratio=1.25):
        power = np.ascontiguousarray(power, np.float64)
        offsets = np.ascontiguousarray(offsets, np.uint32)
        nbr = np.ascontiguousarray(nbr, np.uint32)
        idx = np.zeros(num_sources, np.uint32)
        pw = np.zeros(num_sources)
        low = np.zeros(num_sources, np.uint8)
        cnt = C.c_uint32()
        self._chk(self.L.orc_peaks(_p(power, _f64p), C.c_uint32(power.shape[0]), _p(offsets, _u32p), _p(nbr, _u32p),
                                   C.c_uint32(num_sources), C.c_float(low_power_ratio), _p(idx, _u32p),
                                   _p(pw, _f64p), _p(low, _u8p), C.byref(cnt)))
        c = cnt.value
        return idx[:c].copy(), pw[:c].copy(), low[:c].astype(bool)

    def locate(self, x, k, h, dirs, t, num_sources, floor=1e-12, squared=False, low_power_ratio=1.25,
               radius_deg=10.0, threads=None, keep_bins=False):
        """The FP64 block loop (pipeline.cpp:227-245 with path=reference)."""
        r = self.correlation(x, t)
        off, nbr = self.topology(dirs, radius_deg)
        kinv = np.stack([self.mat_inverse(k[b], bin_label=b) for b in range(k.shape[0])])
        out = dict(power=[], bin_power=[], idx=[], pw=[], low=[], sigma=[])
        for rb in r:
            g = self.gsvd_reference(k, rb, kinv=kinv, threads=threads)
            p, bp = self.spectrum(g["e"], h, num_sources, floor, squared, threads, keep_bins)
            i, pw, lo = self.peaks(p, off, nbr, num_sources, low_power_ratio)
            out["power"].append(p)
            out["bin_power"].append(bp)
            out["idx"].append(i)
            out["pw"].append(pw)
            out["low"].append(lo)
            out["sigma"].append(g["sigma"])
        return out


_ref_singleton = None
_port_singleton = None


def ref() -> _Ref:
    global _ref_singleton
    if _ref_singleton is None:
        _ref_singleton = _Ref()
    return _ref_singleton


def port() -> _Port:
    global _port_singleton
    if _port_singleton is None:
        _port_singleton = _Port()
    return _port_singleton


def ref_available() -> bool:
    return os.path.exists(REF_SO)
