"""Randomized parity sweep: the sm_100a GSVD and MUSIC spectrum against the
FP64 oracle (the C restatement pinned to the reference, oracle/) over random
shapes and inputs — every solver path (the lane-group solver at m <= 16, the
fused CTA solver for other m, the split m = 60 solver), full-rank and
rank-deficient R, exact ties, identity and random noise models, and scales
from 1e-6 to 1e6.

Tolerances as in test_gpu_parity.py: sigma within 1e-9 sigma_max, canonical
vectors within 1e-6, per-bin spectrum within 1e-6 relative (the engine's
spectrum of its own E against the oracle's spectrum of the oracle's E).

SSLG_FUZZ_CASES sets the number of cases (default 40, a few seconds);
SSLG_FUZZ_OUT=<path> writes a JSON summary (worst errors per path).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIGMA_TOL = 1e-9
E_TOL = 1e-6
BINP_TOL = 1e-6
M_CHOICES = [1, 2, 3, 5, 7, 8, 8, 12, 16, 16, 17, 24, 31, 37, 48, 59, 60, 60, 60, 63, 64]


def _case(rng, idx):
    m = int(rng.choice(M_CHOICES))
    bins = int(rng.integers(2, 5))
    kind = ["full", "deficient", "tied", "rank1"][idx % 4]
    scale = float(10.0 ** rng.uniform(-6, 6))
    r = np.empty((bins, m, m), np.complex64)
    for b in range(bins):
        if kind == "tied" and m >= 3:
            d = int(rng.integers(2, max(3, m // 2 + 1)))
            s = np.sort(rng.uniform(0.5, 9.0, m))[::-1].copy()
            i0 = int(rng.integers(0, m - d + 1))
            s[i0:i0 + d] = s[i0]
            s = np.sort(s)[::-1]
            q, _ = np.linalg.qr(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))
            r[b] = (q * s) @ q.conj().T * scale
        else:
            rank = {"full": m, "deficient": max(1, m // 2), "rank1": 1}.get(kind, m)
            x = rng.standard_normal((m, rank)) + 1j * rng.standard_normal((m, rank))
            r[b] = (x @ x.conj().T / rank * scale).astype(np.complex64)
    if rng.random() < 0.5:
        k = np.broadcast_to(np.eye(m, dtype=np.complex64), (bins, m, m)).copy()
        kname = "identity"
    else:
        kb = rng.standard_normal((bins, m, m)) + 1j * rng.standard_normal((bins, m, m))
        k = (kb @ kb.conj().transpose(0, 2, 1) / m + 0.5 * np.eye(m)).astype(np.complex64)
        kname = "random"
    return m, bins, kind, kname, scale, r, k


def _path(m):
    return "lane-group" if m <= 16 else ("split-60" if m == 60 else "fused-cta")


def test_randomized_parity_against_oracle(port):
    from paper_2504_03373_b200 import ssl, synth

    n = int(os.environ.get("SSLG_FUZZ_CASES", "40"))
    rng = np.random.default_rng(20261017)
    worst = {}
    failures = []
    for idx in range(n):
        m, bins, kind, kname, scale, r, k = _case(rng, idx)
        ns = max(0, min(2, m - 1))
        kw = {"music": ssl.MusicConfig(num_sources=ns)} if ns > 0 else {}
        eng = ssl.Engine(m, bins, window_frames=2, max_batch=2, **kw)
        eng.set_noise_model(k)
        sigma, e, _, conv = eng.gsvd(r)
        want = port.gsvd_reference(k, r, threads=4)
        smax = np.maximum(want["sigma"][:, :1], 1e-300)
        es = float(np.max(np.abs(sigma[0] - want["sigma"]) / smax))
        ee = float(np.max(np.abs(e[0] - want["e"])))
        ep = 0.0
        if ns > 0:
            dirs = synth.azimuth_grid(30.0)
            h = synth.steering(synth.circular(m, 0.05), dirs, 10, 10 + bins - 1)
            eng.set_steering(h, dirs)
            _, bp = eng.spectrum(e)
            _, bpw = port.spectrum(want["e"], h, ns, keep_bins=True)
            ep = float(np.max(np.abs(bp[0] - bpw) / np.abs(bpw)))
        eng.close()
        ok = bool(np.all(conv) == bool(np.all(want["conv"]))) and es <= SIGMA_TOL and ee <= E_TOL and ep <= BINP_TOL
        key = _path(m)
        w = worst.setdefault(key, {"cases": 0, "sigma": 0.0, "e": 0.0, "bin_power": 0.0})
        w["cases"] += 1
        w["sigma"] = max(w["sigma"], es)
        w["e"] = max(w["e"], ee)
        w["bin_power"] = max(w["bin_power"], ep)
        if not ok:
            failures.append(dict(case=idx, m=m, bins=bins, kind=kind, k=kname, scale=scale, sigma=es, e=ee,
                                 bin_power=ep))
    out = os.environ.get("SSLG_FUZZ_OUT")
    if out:
        with open(out, "w") as f:
            json.dump({"cases": n, "seed": 20261017, "tolerances": {"sigma_rel_sigma_max": SIGMA_TOL,
                                                                    "e_abs": E_TOL, "bin_power_rel": BINP_TOL},
                       "worst_by_path": worst, "failures": failures}, f, indent=1)
    assert not failures, failures[:5]
