"""Engine runs for compute-sanitizer (development aid), one case per path:

  python tools/sanitize.py CASE        (under compute-sanitizer --tool memcheck|racecheck|synccheck)
  cases: c1 c3 corners stream small tc er formats all

  c1       the 8-channel pipeline on the c1_band fixture
  c3       60-channel flagship kernels on a few bins, short windows (big_vanish), DMMA spectrum
  corners  generic canonical kernel (refine mode, a tied group above kZMax), rejected picker
           candidates, generic m = 37 and m = 16
  stream   device STFT, sample pushes across calls, async pushes with the result ring, the gate
  small    the lane-group solver (m = 8 and 16) incl. in-group canonicalization of vanishing / tied
           bins and the refine-mode worklist
  tc       the tcgen05 spectrum (bulk copies, TMEM, mbarriers) with padding and odd m
  er       E_r / residual, inverses (float, pivot-free), PD gate eigenvalues
  formats  noise capture, file loaders into a context, the direct-sum STFT
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_03373_b200 import formats, ssl, synth  # noqa: E402
from paper_2504_03373_b200.errors import NumericalError, ValidationError  # noqa: E402


def golden(name):
    return dict(np.load(os.path.join(ROOT, "tests", "golden", name + ".npz")))


def case_c1():
    g = golden("c1_band")
    t, ns = int(g["t"]), int(g["ns"])
    m, bins = g["x"].shape[1], g["x"].shape[2]
    eng = ssl.Engine(m, bins, window_frames=t, music=ssl.MusicConfig(num_sources=ns), max_batch=16)
    eng.set_noise_model(g["k"])
    eng.set_steering(g["h"], g["dirs"])
    out = eng.push(g["x"], want_power=True)
    print("c1 blocks", out["n"], "power rel", np.max(np.abs(out["power"] - g["power"]) / g["power"]))


def case_c3():
    w = synth.make("c3", frames=40)
    sl = slice(100, 104)
    for t in (24, 30):
        eng = ssl.Engine(60, 4, window_frames=t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=4)
        eng.set_noise_model(np.ascontiguousarray(w.k[sl]))
        eng.set_steering(np.ascontiguousarray(w.h[:, sl]), w.dirs)
        out = eng.push(np.ascontiguousarray(w.x[:t + 2, :, sl]), want_power=True)
        print("c3 T", t, "blocks", out["n"], "idx", out["idx"].tolist())
        eng.close()


def _gsvd(m, r, k, solver=None):
    eng = ssl.Engine(m, r.shape[0], window_frames=2, max_batch=2, solver=solver)
    eng.set_noise_model(k)
    sigma, e, _, conv = eng.gsvd(r)
    eng.close()
    return sigma, conv


def case_corners():
    rng = np.random.default_rng(3)
    m, bins = 60, 2
    eye = np.broadcast_to(np.eye(m, dtype=np.complex64), (bins, m, m)).copy()
    s = np.concatenate([np.linspace(9.0, 5.0, 10), np.full(30, 2.0), np.linspace(1.5, 0.5, 20)])
    r = np.empty((bins, m, m), np.complex64)
    for b in range(bins):
        q, _ = np.linalg.qr(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))
        r[b] = (q * s) @ q.conj().T
    print("tied30", _gsvd(m, r, eye)[1].all())
    x = rng.standard_normal((bins, m, 30)) + 1j * rng.standard_normal((bins, m, 30))
    x[:, 0, 2:] = 0
    x[:, 2, 2:] = 0
    x[:, :, :2] = 0
    x[:, 0, 0] = 3.0
    x[:, 2, 1] = 2.0
    r2 = (x @ x.conj().transpose(0, 2, 1) / 30).astype(np.complex64)
    print("reject", _gsvd(m, r2, eye)[1].all())
    print("refine", _gsvd(m, r2, eye, ssl.SolverConfig(refine_leading=True))[1].all())
    for mm in (37, 16):
        xb = rng.standard_normal((bins, mm, mm // 2)) + 1j * rng.standard_normal((bins, mm, mm // 2))
        rr = (xb @ xb.conj().transpose(0, 2, 1)).astype(np.complex64)
        kk = np.broadcast_to(np.eye(mm, dtype=np.complex64), (bins, mm, mm)).copy()
        print("m", mm, _gsvd(mm, rr, kk)[1].all())


def case_stream():
    g = np.load(os.path.join(ROOT, "tests", "golden", "stft.npz"))
    fl, sh, win, b0, b1 = (int(v) for v in g["hann_band_cfg"])
    stft = ssl.StftConfig(fl, sh, "hann", b0, b1)
    audio = g["hann_band_audio"]
    m = audio.shape[0]
    eng = ssl.Engine(m, stft.bin_count(), window_frames=6, music=ssl.MusicConfig(num_sources=2), max_batch=8)
    rng = np.random.default_rng(1)
    a = rng.standard_normal((stft.bin_count(), m, m)) + 1j * rng.standard_normal((stft.bin_count(), m, m))
    eng.set_noise_model((a @ a.conj().transpose(0, 2, 1) / m + np.eye(m)).astype(np.complex64))
    dirs = synth.azimuth_grid(5.0)
    eng.set_steering(synth.steering(synth.circular(m, 0.05), dirs, stft.bin_min, stft.bin_max, stft.frame_length),
                     dirs)
    eng.set_stft(stft)
    o = eng.push_samples(audio[:, :1500], want_power=True)
    o2 = eng.push_samples(audio[:, 1500:], want_power=True)
    print("sync blocks", o["n"] + o2["n"])
    eng.reset_window()
    tickets = [eng.push_samples_async(audio[:, s:s + 700]) for s in range(0, audio.shape[1], 700)]
    print("async blocks", eng.wait_results(tickets[-1])["n"])
    eng.reset_window()
    bad = audio.copy()
    bad[1, 2500] = np.nan
    t1 = eng.push_samples_async(bad[:, :2000])
    t2 = eng.push_samples_async(bad[:, 2000:])
    eng.wait_results(t1)
    try:
        eng.wait_results(t2)
        print("gate FAILED")
    except ValidationError:
        print("gate ok")
    eng.close()


def case_small():
    w = synth.make("c1", frames=58)
    eng = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=16)
    eng.set_noise_model(w.k)
    eng.set_steering(w.h, w.dirs)
    out = eng.push(w.x, want_power=True)
    print("small blocks", out["n"])
    # worklisted bins: an exactly repeated value and a rank-deficient bin
    rng = np.random.default_rng(5)
    r = np.zeros((3, 8, 8), np.complex64)
    r[0] = 2.0 * np.eye(8)
    x = rng.standard_normal((8, 3)) + 1j * rng.standard_normal((8, 3))
    r[1] = x @ x.conj().T
    r[2] = np.diag(np.arange(1, 9)).astype(np.complex64)
    eng2 = ssl.Engine(8, 3, window_frames=2, max_batch=2)
    eng2.set_noise_identity()
    print("small canonical groups", eng2.gsvd(r)[3].all())
    eng.close()
    eng2.close()
    # m = 16 (16-lane groups): a tied pair, a rank-deficient bin, refine mode (worklist)
    r16 = np.zeros((3, 16, 16), np.complex64)
    r16[0] = np.diag(np.r_[3.0, 3.0, np.arange(14, 0, -1)]).astype(np.complex64)
    x16 = rng.standard_normal((16, 5)) + 1j * rng.standard_normal((16, 5))
    r16[1] = x16 @ x16.conj().T
    r16[2] = np.diag(np.arange(16, 0, -1)).astype(np.complex64)
    for refine in (False, True):
        eng3 = ssl.Engine(16, 3, window_frames=2, max_batch=2, solver=ssl.SolverConfig(refine_leading=refine))
        eng3.set_noise_identity()
        print("small m=16 refine", refine, eng3.gsvd(r16)[3].all())
        eng3.close()


def case_tc():
    rng = np.random.default_rng(9)
    for m, ns, dirs in ((13, 2, 300), (60, 3, 1368)):
        bins = 3
        h = (rng.standard_normal((dirs, bins, m)) + 1j * rng.standard_normal((dirs, bins, m))).astype(np.complex64)
        e = np.linalg.qr(rng.standard_normal((bins, m, m)) + 1j * rng.standard_normal((bins, m, m)))[0]
        eng = ssl.Engine(m, bins, window_frames=1, music=ssl.MusicConfig(num_sources=ns), max_batch=2)
        eng.set_steering(h, np.stack([np.arange(dirs) * 0.25, np.zeros(dirs)], 1))
        eng.set_spectrum_path(1)
        p, _ = eng.spectrum(np.stack([e, e]))
        print("tc m", m, "dirs", dirs, "finite", bool(np.all(np.isfinite(p))))
        eng.close()


def case_er():
    rng = np.random.default_rng(4)
    m = 12
    r = (rng.standard_normal((2, m, m)) + 1j * rng.standard_normal((2, m, m))).astype(np.complex64)
    x = rng.standard_normal((m, 4)) + 1j * rng.standard_normal((m, 4))
    r[1] = (x @ x.conj().T).astype(np.complex64)  # rank deficient: vanishing rows
    k = np.broadcast_to(np.eye(m, dtype=np.complex64), (2, m, m)).copy()
    eng = ssl.Engine(m, 2, window_frames=2, max_batch=2, solver=ssl.SolverConfig(compute_residual=True))
    eng.set_noise_model(k, check_pd=True)
    sig, e, sw, cv, er, res = eng.gsvd(r[None], want_er=True, want_resid=True)
    print("er residual", res.tolist())
    print("inverse f", eng.noise_inverse(0).shape)
    eng.close()
    bad = k.copy()
    bad[1, 0, 0] = -1.0
    eng = ssl.Engine(m, 2, window_frames=2, max_batch=2, solver=ssl.SolverConfig(pivoting="none"))
    try:
        eng.set_noise_model(bad, check_pd=True)
    except NumericalError as exc:
        print("pd gate:", exc)
    eng.close()


def case_formats():
    g = np.load(os.path.join(ROOT, "tests", "golden", "stft.npz"))
    audio = g["hann_480_audio"]
    fl, sh, win, b0, b1 = (int(v) for v in g["hann_480_cfg"])
    stft = ssl.StftConfig(fl, sh, "hann", b0, b1)
    eng = ssl.Engine(audio.shape[0], stft.bin_count(), max_batch=4)
    eng.set_stft(stft)
    fr = eng.stft(audio)
    print("dft frames equal", np.array_equal(fr.view(np.uint32), g["hann_480_frames"].view(np.uint32)))
    noise = np.random.default_rng(2).standard_normal((audio.shape[0], 6000)).astype(np.float32)
    k = eng.capture_noise_model(noise)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "k.sslc")
        formats.save_correlation(p, k, 10)
        eng.load_noise_model(p)
    print("capture + load ok", k.shape)
    eng.close()


CASES = {"c1": case_c1, "c3": case_c3, "corners": case_corners, "stream": case_stream, "small": case_small,
         "tc": case_tc, "er": case_er, "formats": case_formats}

if __name__ == "__main__":
    names = sys.argv[1:] or ["all"]
    if names == ["all"]:
        names = list(CASES)
    for n in names:
        CASES[n]()
