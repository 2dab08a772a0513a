"""GPU parity at the paper's array size (BASELINE configs[2], C3: 60 channels,
257 bins, 72 azimuths, T = 50 < M so every block has a 10-dimensional
vanishing subspace) and on the C4 az x el grid (1368 directions, 3 sources,
exact steering ties at the poles).

The scenes come from the seeded synthetic generator (synth.py); the checker is
the C restatement of the reference's FP64 path (oracle/sslref.c, pinned bit for
bit to the compiled reference by tests/test_oracle.py).  Tolerances are the
ones of test_gpu_parity.py:
  sigma       |d sigma| <= 1e-9 sigma_max
  P(theta,w)  relative <= 1e-6
  Pbar(theta) relative <= 1e-8
  peaks       identical indices and low-power flags
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIGMA_TOL = 1e-9
BINP_TOL = 1e-6
PBAR_TOL = 1e-8


def _run(config, frames, port, max_batch=8, spectrum_path=0):
    from paper_2504_03373_b200 import ssl, synth

    w = synth.make(config, frames=frames)
    eng = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=max_batch)
    eng.set_noise_model(w.k)
    eng.set_steering(w.h, w.dirs)
    eng.set_spectrum_path(spectrum_path)
    out = eng.push(w.x, want_power=True)
    n = out["n"]
    res = eng.read_results(min(n, max_batch), power=True, bin_power=True, sigma=True)
    eng.close()
    want = port.locate(w.x, w.k, w.h, w.dirs, w.t, w.ns, keep_bins=True, threads=os.cpu_count())
    return w, out, res, want


def _check(out, res, want, pbar_tol=PBAR_TOL, binp_tol=BINP_TOL):
    n = out["n"]
    assert n == len(want["power"])
    for b in range(n):
        rel = np.max(np.abs(out["power"][b] - want["power"][b]) / np.abs(want["power"][b]))
        assert rel <= pbar_tol, (b, rel)
        c = int(out["count"][b])
        assert c == len(want["idx"][b])
        assert np.array_equal(out["idx"][b][:c], want["idx"][b])
        assert np.array_equal(out["low"][b][:c].astype(bool), want["low"][b])
    k0 = n - res["power"].shape[0]
    for j in range(res["power"].shape[0]):
        smax = want["sigma"][k0 + j][:, :1]
        assert np.max(np.abs(res["sigma"][j] - want["sigma"][k0 + j]) / smax) <= SIGMA_TOL
        ref = want["bin_power"][k0 + j]
        assert np.max(np.abs(res["bin_power"][j] - ref) / np.abs(ref)) <= binp_tol
    assert np.all(res["conv"])


def test_c3_blocks_against_oracle(port):
    w, out, res, want = _run("c3", 53, port)
    assert out["n"] == 4
    _check(out, res, want)
    # the scene's two targets are the two reported sources
    assert set(out["idx"][0][:2].tolist()) == set(w.targets)


@pytest.mark.parametrize("path", [0, 1], ids=["fp64", "tcgen05"])
def test_c4_azel_grid_against_oracle(port, path):
    """Both spectrum kernels on the 1368-direction grid: the FP64 one at the
    FP64 tolerances, the tcgen05 tf32x3 one (the default for grids this
    large) at its stated ones (tests/test_gpu_spectrum_tc.py)."""
    w, out, res, want = _run("c4", 51, port, spectrum_path=path)
    assert w.h.shape[0] == 72 * 19
    if path == 0:
        _check(out, res, want)
    else:
        _check(out, res, want, pbar_tol=5e-7, binp_tol=1e-6)
