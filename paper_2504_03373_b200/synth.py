"""Synthetic STFT-domain workloads for the bench (BASELINE.json configs).

Builds, directly in the frequency domain, the inputs the hot path consumes:
spectrum frames X [F][m][bins] (SpectrumFrame layout), a noise correlation K
captured from noise-only frames, and the far-field steering table H
[dirs][bins][m].  The array geometries, direction grids and steering formula
follow the reference generators (ArrayGeometry::circular / spherical,
azimuth_grid, make_steering: proj/src/synth.cpp:59-149) — computed in FP64,
stored FP32 — so the GSVD sees the same structure as the reference's scenes
(rank <= T correlation windows, directional rotor noise, diffuse floor).
This is input tooling for measurement, not part of the hot path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

SPEED_OF_SOUND = 343.0


def circular(count: int, radius: float) -> np.ndarray:
    ang = 2.0 * np.pi * np.arange(count) / count
    return np.stack([radius * np.cos(ang), radius * np.sin(ang), np.zeros(count)], 1)


def spherical(count: int, radius: float) -> np.ndarray:
    ga = np.pi * (3.0 - np.sqrt(5.0))
    i = np.arange(count, dtype=np.float64)
    z = 1.0 - 2.0 * (i + 0.5) / count
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    az = i * ga
    return np.stack([radius * r * np.cos(az), radius * r * np.sin(az), radius * z], 1)


def azimuth_grid(step_deg: float = 5.0) -> np.ndarray:
    n = int(np.floor(360.0 / step_deg + 1e-9))
    return np.stack([np.arange(n) * step_deg, np.zeros(n)], 1)


def azel_grid(step_deg: float = 5.0, el_min=-90.0, el_max=90.0, el_step=10.0) -> np.ndarray:
    ring = azimuth_grid(step_deg)
    els = np.arange(el_min, el_max + 1e-9, el_step)
    return np.concatenate([np.stack([ring[:, 0], np.full(len(ring), e)], 1) for e in els], 0)


def unit(dirs_deg: np.ndarray) -> np.ndarray:
    az = np.deg2rad(dirs_deg[:, 0])
    el = np.deg2rad(dirs_deg[:, 1])
    return np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)], 1)


def steering(mics: np.ndarray, dirs_deg: np.ndarray, bin_min: int, bin_max: int, frame_length: int = 512,
             sample_rate: int = 16000) -> np.ndarray:
    """[dirs][bins][m] complex64: exp(-j 2 pi f tau), tau = -(u.p)/c (synth.cpp:17-22)."""
    u = unit(dirs_deg)
    tau = -(u @ mics.T) / SPEED_OF_SOUND  # [dirs][m]
    f = np.arange(bin_min, bin_max + 1, dtype=np.float64) * sample_rate / frame_length
    ang = -2.0 * np.pi * f[None, :, None] * tau[:, None, :]
    return (np.cos(ang) + 1j * np.sin(ang)).astype(np.complex64)


@dataclass
class Workload:
    name: str
    x: np.ndarray  # [F][m][bins] complex64
    k: np.ndarray  # [bins][m][m] complex64
    h: np.ndarray  # [dirs][bins][m] complex64
    dirs: np.ndarray  # [dirs][2]
    t: int
    ns: int
    targets: List[int] = field(default_factory=list)

    @property
    def m(self):
        return self.x.shape[1]

    @property
    def bins(self):
        return self.x.shape[2]


def _field(rng, mics, src_dirs, levels_db, bins_idx, frames, frame_length, sample_rate, diffuse_db):
    m = mics.shape[0]
    nb = len(bins_idx)
    x = np.zeros((frames, nb, m), np.complex128)
    if len(src_dirs):
        hs = steering(mics, np.asarray(src_dirs, np.float64), bins_idx[0], bins_idx[-1], frame_length,
                      sample_rate).astype(np.complex128)  # [S][bins][m]
        for s, lvl in enumerate(levels_db):
            amp = 10 ** (lvl / 20.0) * np.sqrt(frame_length / 2.0)
            g = (rng.standard_normal((frames, nb)) + 1j * rng.standard_normal((frames, nb))) * (amp / np.sqrt(2))
            x += g[:, :, None] * hs[s][None]
    if diffuse_db is not None:
        amp = 10 ** (diffuse_db / 20.0) * np.sqrt(frame_length / 2.0)
        x += (rng.standard_normal((frames, nb, m)) + 1j * rng.standard_normal((frames, nb, m))) * (amp / np.sqrt(2))
    return x


def drone_scene(name: str = "c3", m: int = 60, geometry: str = "circular", radius: float = 0.3,
                bin_min: int = 0, bin_max: int = 256, dirs: np.ndarray = None, frames: int = 400, t: int = 50,
                ns: int = 2, targets_deg: Sequence[float] = (40.0, 150.0), target_db: float = -3.0,
                rotors_deg: Sequence[float] = (45.0, 135.0, 225.0, 315.0), rotor_db: float = 0.0,
                diffuse_db: float = -20.0, noise_frames: int = 240, seed: int = 11, frame_length: int = 512,
                sample_rate: int = 16000) -> Workload:
    """Low-SNR drone-like scene (BASELINE configs 3-5): targets below four
    rotor noise sources plus a diffuse floor; K is captured from noise-only
    frames (the capture_noise_model procedure, synth.cpp:329-373)."""
    rng = np.random.default_rng(seed)
    mics = circular(m, radius) if geometry == "circular" else spherical(m, radius)
    dirs = azimuth_grid(5.0) if dirs is None else dirs
    bins_idx = np.arange(bin_min, bin_max + 1)
    src = [(a, 0.0) for a in targets_deg] + [(a, 0.0) for a in rotors_deg]
    lv = [target_db] * len(targets_deg) + [rotor_db] * len(rotors_deg)
    x = _field(rng, mics, src, lv, bins_idx, frames, frame_length, sample_rate, diffuse_db)
    noise = _field(rng, mics, [(a, 0.0) for a in rotors_deg], [rotor_db] * len(rotors_deg), bins_idx,
                   noise_frames, frame_length, sample_rate, diffuse_db)
    # K = mean x x^H over the noise-only frames, FP64 then narrowed
    k = np.einsum("fbi,fbj->bij", noise, noise.conj()) / noise_frames
    k = k.astype(np.complex64)
    h = steering(mics, dirs, bin_min, bin_max, frame_length, sample_rate)
    xs = np.ascontiguousarray(x.transpose(0, 2, 1)).astype(np.complex64)  # [F][m][bins]
    tgt = [int(np.argmin(np.abs(dirs[:, 0] - a) + np.abs(dirs[:, 1]))) for a in targets_deg]
    return Workload(name, xs, k, h, np.ascontiguousarray(dirs, np.float64), t, ns, tgt)


CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": dict(m=8, radius=0.05, targets_deg=(40.0, 150.0), target_db=0.0, rotors_deg=(), diffuse_db=-20.0, ns=2),
    # C2: K from random_noise_model(16, 257, seed) as bench.cpp:178-206
    "c2": dict(m=16, radius=0.05, targets_deg=(75.0, 200.0), target_db=0.0, rotors_deg=(300.0,), ns=2,
               noise_model="random"),
    # targets at 0 dB each under four rotors at -10 dB each (-4 dB total) and a
    # -20 dB diffuse floor: ~ +4 dB per target against the whole noise field
    "c3": dict(m=60, radius=0.3, ns=2, target_db=0.0, rotor_db=-10.0),
    "c4": dict(m=60, radius=0.3, ns=3, targets_deg=(40.0, 150.0, 260.0), target_db=0.0, rotor_db=-10.0),
}


def make(config: str, frames: int = 400, seed: int = 11) -> Workload:
    kw = dict(CONFIGS[config])
    random_k = kw.pop("noise_model", "captured") == "random"
    if config == "c4":
        kw["dirs"] = azel_grid(5.0)
    w = drone_scene(name=config, frames=frames, seed=seed, **kw)
    if random_k:
        w.k = random_noise_model(w.m, w.bins, seed)
    return w


# ---------------------------------------------------------------------------
# time-domain scenes (SampleBlock input for the STFT front end)
# ---------------------------------------------------------------------------


@dataclass
class PcmWorkload:
    name: str
    pcm: np.ndarray  # [m][samples] float32 (SampleBlock::channels)
    k: np.ndarray  # [bins][m][m] complex64
    h: np.ndarray  # [dirs][bins][m] complex64
    dirs: np.ndarray  # [dirs][2]
    t: int
    ns: int
    bin_min: int
    bin_max: int
    frame_length: int = 512
    shift: int = 160
    targets: List[int] = field(default_factory=list)

    @property
    def m(self):
        return self.pcm.shape[0]

    @property
    def bins(self):
        return self.bin_max - self.bin_min + 1


def _pcm_field(rng, mics, src_dirs, levels_db, n, sample_rate, diffuse_db):
    """Far-field white sources delayed per microphone by tau = -(u . p) / c
    (the make_steering convention, synth.cpp:123-149: mic spectrum = S(f)
    exp(-j 2 pi f tau)), applied as an exact frequency-domain delay over the
    whole signal, plus an independent diffuse floor per microphone."""
    m = mics.shape[0]
    f = np.fft.rfftfreq(n, 1.0 / sample_rate)
    x = np.zeros((m, n))
    if len(src_dirs):
        u = unit(np.asarray(src_dirs, np.float64))  # [S][3]
        tau = -(u @ mics.T) / SPEED_OF_SOUND  # [S][m]
        for s, lvl in enumerate(levels_db):
            spec = np.fft.rfft(rng.standard_normal(n) * 10 ** (lvl / 20.0))
            x += np.fft.irfft(spec[None, :] * np.exp(-2j * np.pi * f[None, :] * tau[s][:, None]), n)
    if diffuse_db is not None:
        x += rng.standard_normal((m, n)) * 10 ** (diffuse_db / 20.0)
    return x


def _stft_np(x, frame_length, shift, bin_min, bin_max):
    """Periodic-Hann STFT (numpy; used only to capture K from noise-only PCM)."""
    w = 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(frame_length) / frame_length)
    nf = (x.shape[1] - frame_length) // shift + 1
    idx = np.arange(frame_length)[None, :] + shift * np.arange(nf)[:, None]
    fr = np.fft.rfft(x[:, idx] * w[None, None, :], axis=2)[:, :, bin_min:bin_max + 1]  # [m][F][bins]
    return fr.transpose(1, 2, 0)  # [F][bins][m]


def drone_scene_pcm(name: str = "c3", m: int = 60, radius: float = 0.3, bin_min: int = 0, bin_max: int = 256,
                    dirs: np.ndarray = None, duration_s: float = 2.0, t: int = 50, ns: int = 2,
                    targets_deg: Sequence[float] = (40.0, 150.0), target_db: float = -3.0,
                    rotors_deg: Sequence[float] = (45.0, 135.0, 225.0, 315.0), rotor_db: float = 0.0,
                    diffuse_db: float = -20.0, noise_s: float = 2.5, seed: int = 11, frame_length: int = 512,
                    shift: int = 160, sample_rate: int = 16000) -> PcmWorkload:
    """The C3 drone scene as PCM: targets under four rotor sources and a
    diffuse floor; K captured from a separate noise-only recording
    (capture_noise_model, synth.cpp:329-373)."""
    rng = np.random.default_rng(seed)
    mics = circular(m, radius)
    dirs = azimuth_grid(5.0) if dirs is None else dirs
    src = [(a, 0.0) for a in targets_deg] + [(a, 0.0) for a in rotors_deg]
    lv = [target_db] * len(targets_deg) + [rotor_db] * len(rotors_deg)
    n = int(duration_s * sample_rate)
    pcm = _pcm_field(rng, mics, src, lv, n, sample_rate, diffuse_db).astype(np.float32)
    noise = _pcm_field(rng, mics, [(a, 0.0) for a in rotors_deg], [rotor_db] * len(rotors_deg),
                       int(noise_s * sample_rate), sample_rate, diffuse_db)
    fr = _stft_np(noise, frame_length, shift, bin_min, bin_max)
    k = (np.einsum("fbi,fbj->bij", fr, fr.conj()) / fr.shape[0]).astype(np.complex64)
    h = steering(mics, dirs, bin_min, bin_max, frame_length, sample_rate)
    tgt = [int(np.argmin(np.abs(dirs[:, 0] - a) + np.abs(dirs[:, 1]))) for a in targets_deg]
    return PcmWorkload(name, pcm, k, h, np.ascontiguousarray(dirs, np.float64), t, ns, bin_min, bin_max,
                       frame_length, shift, tgt)


def make_pcm(config: str, duration_s: float = 2.0, seed: int = 11) -> PcmWorkload:
    kw = dict(CONFIGS[config])
    kw.pop("geometry", None)
    random_k = kw.pop("noise_model", "captured") == "random"
    if config == "c4":
        kw["dirs"] = azel_grid(5.0)
    w = drone_scene_pcm(name=config, duration_s=duration_s, seed=seed, **kw)
    if random_k:
        w.k = random_noise_model(w.m, w.bins, seed)
    return w


def describe(config: str) -> str:
    """One-line description of a bench scene (the JSON line's workload)."""
    kw = CONFIGS[config]
    m, r = kw["m"], kw["radius"]
    tg = kw.get("targets_deg", (40.0, 150.0))
    rot = kw.get("rotors_deg", (45.0, 135.0, 225.0, 315.0))
    tdb = kw.get("target_db", -3.0)
    rdb = kw.get("rotor_db", 0.0)
    dif = kw.get("diffuse_db", -20.0)
    grid = "72 az x 19 el (1368 directions)" if config == "c4" else "72 azimuths"
    srcs = f"{len(tg)} targets at {'/'.join(f'{a:g}' for a in tg)} deg ({tdb:g} dB)"
    if rot:
        srcs += f" + {len(rot)} rotor noise source(s) at {'/'.join(f'{a:g}' for a in rot)} deg ({rdb:g} dB)"
    srcs += f" + diffuse ({dif:g} dB)"
    k = ("K = random_noise_model(m, 257, seed) (bench.cpp:178-186)" if kw.get("noise_model") == "random"
         else "K captured from a separate noise-only recording")
    return (f"{m}-ch circular r={r:g} m, 16 kHz, 512-pt FFT, 257 bins, {grid}, {srcs}, {k}, "
            f"T=50, Ns={kw['ns']}")


# ---------------------------------------------------------------------------
# random_noise_model (BASELINE configs[1], "C2": GSVD-MUSIC with synthetic K)
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1


class _MT19937_64:
    """std::mt19937_64 (its output sequence is pinned by the C++ standard;
    the reference draws every synthetic value from it, rng.hpp:1-34)."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _M64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt = np.array(mt, np.uint64)
        self.buf = None
        self.pos = 312

    def _twist(self):
        mt = self.mt
        um, lm = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
        a = np.uint64(0xB5026F5AA96619E9)
        one = np.uint64(1)
        for i in range(312):  # sequential dependence on updated words
            x = (mt[i] & um) | (mt[(i + 1) % 312] & lm)
            xa = x >> one
            if x & one:
                xa ^= a
            mt[i] = mt[(i + 156) % 312] ^ xa
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.buf = [int(v) for v in y]
        self.pos = 0

    def __call__(self) -> int:
        if self.pos >= 312:
            self._twist()
        v = self.buf[self.pos]
        self.pos += 1
        return v


def mix_seed(base: int, tag: int) -> int:
    """ssl::mix_seed (rng.hpp:17-24)."""
    x = (base ^ ((0x632BE59BD9B4E019 * (tag + 1)) & _M64)) & _M64
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _gaussian(g: _MT19937_64) -> float:
    """ssl::gaussian (rng.hpp:27-33): Box-Muller on two 53-bit uniforms,
    through the C library's log/cos like the reference."""
    import math

    u1 = 1.0 - float(g() >> 11) * 2.0 ** -53
    u2 = float(g() >> 11) * 2.0 ** -53
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def random_psd(m: int, g: _MT19937_64, ridge: float) -> np.ndarray:
    """random_psd (bench.cpp:161-176): A A^H / m in FP64 with the reference
    matmul's k-ascending accumulation (mat.hpp:31-44), narrowed to FP32, plus
    `ridge` on the diagonal in float, then the lower triangle mirrored."""
    ar = np.empty((m, m))
    ai = np.empty((m, m))
    for i in range(m):
        for j in range(m):
            # cdouble(gaussian(rng), gaussian(rng)): GCC evaluates the two
            # constructor arguments right to left, so the imaginary part draws first
            ai[i, j] = _gaussian(g)
            ar[i, j] = _gaussian(g)
    # p(i, j) = sum_k a(i, k) * conj(a(j, k)), k ascending; skip exact zeros
    pr = np.zeros((m, m))
    pi = np.zeros((m, m))
    for k in range(m):
        xr, xi = ar[:, k][:, None], ai[:, k][:, None]  # a(i, k)
        yr, yi = ar[:, k][None, :], -ai[:, k][None, :]  # conj(a(j, k)) = b(k, j)
        nz = (xr != 0) | (xi != 0)
        pr = np.where(nz, pr + (xr * yr - xi * yi), pr)
        pi = np.where(nz, pi + (xr * yi + xi * yr), pi)
    inv = 1.0 / float(m)
    out = ((pr * inv).astype(np.float32) + 1j * (pi * inv).astype(np.float32)).astype(np.complex64)
    d = np.arange(m)
    out[d, d] = (out[d, d].real + np.float32(ridge)) + 1j * out[d, d].imag
    iu = np.triu_indices(m, 1)
    out[iu[1], iu[0]] = np.conj(out[iu])
    return out


def random_noise_model(m: int, bins: int, seed: int) -> np.ndarray:
    """random_noise_model (bench.cpp:178-186): K [bins][m][m] cf32, every bin
    Hermitian positive definite (ridge 0.5), one mt19937_64 stream per bin
    seeded mix_seed(seed, 0x4b00 + b)."""
    return np.stack([random_psd(m, _MT19937_64(mix_seed(seed, 0x4B00 + b)), 0.5) for b in range(bins)])
