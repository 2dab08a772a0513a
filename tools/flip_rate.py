"""Canonicalization flip-rate report (SURVEY §7 hard part 2; VERDICT r01
"what's weak" 1): over a long C3 stream rendered by the reference's own
generators, how often do the discrete decisions of canonicalize_subspaces
(gsvd.cpp:381-565) -- the vanishing count z (values <= 1e-5 sigma_max) and the
tie-group partition of the kept values (consecutive gaps <= 1e-5 sigma_max)
-- come out differently in this engine than in the reference's FP64 path
(gsvd_reference), and how often the reference's own float path (gsvd)
disagrees with its FP64 path on the same blocks.  Also the broadband-power
error and peak agreement of the engine against the FP64 path on every block.

  python tools/flip_rate.py [--blocks 200] [--out profiles/r02/flip_rate.json]

Needs a GPU and oracle/_ref (the compiled reference).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def structure(sigma):
    """(z, tie-group sizes of the kept values) per gsvd.cpp:475-497."""
    smax = sigma[0] if sigma[0] > 0 else 0.0
    gap = 1e-5 * smax
    m = len(sigma)
    z = 0
    while z < m and sigma[m - 1 - z] <= gap:
        z += 1
    lead = m - z
    groups = []
    i = 0
    while i < lead:
        end = i
        while end + 1 < lead and sigma[end] - sigma[end + 1] <= gap:
            end += 1
        groups.append(end - i + 1)
        i = end + 1
    return z, tuple(groups)


def main():
    import oracle
    from paper_2504_03373_b200 import ssl

    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=200)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "flip_rate.json"))
    args = ap.parse_args()
    t, ns, nb = 50, 2, args.blocks
    rotors = [oracle.Source(a, level_db=0.0, noise_role=True) for a in (45.0, 135.0, 225.0, 315.0)]
    sc = oracle.Scene(mics=60, radius=0.3, duration_s=((t - 1 + nb - 1) * 160 + 512) / 16000.0 + 1e-6, seed=11,
                      diffuse_db=-20.0, bin_min=0, bin_max=256,
                      sources=[oracle.Source(40.0), oracle.Source(150.0)] + rotors, noise="captured",
                      noise_duration_s=2.0)
    R = oracle.ref()
    P = oracle.port()
    t0 = time.time()
    w = R.workload(sc)
    print(f"scene: {w.x.shape} frames x ch x bins, {time.time() - t0:.1f}s", flush=True)

    # the engine, 40 blocks per push
    eng = ssl.Engine(w.m, w.bins, window_frames=t, music=ssl.MusicConfig(num_sources=ns), max_batch=40)
    eng.set_noise_model(w.k)
    eng.set_steering(w.h, w.dirs)
    eng.push(w.x[: t - 1])
    sig, pw, idx = [], [], []
    for f0 in range(t - 1, t - 1 + nb, 40):
        n = min(40, t - 1 + nb - f0)
        out = eng.push(w.x[f0:f0 + n], want_power=True)
        res = eng.read_results(out["n"], sigma=True)
        sig.extend(res["sigma"])
        pw.extend(out["power"])
        idx.extend([out["idx"][b][: out["count"][b]] for b in range(out["n"])])
    eng.close()
    print(f"engine: {len(sig)} blocks, {time.time() - t0:.1f}s", flush=True)

    # the reference's FP64 path (restatement pinned bit for bit to it)
    want = P.locate(w.x[: t - 1 + nb], w.k, w.h, w.dirs, t, ns, threads=os.cpu_count())
    print(f"FP64 reference path: {time.time() - t0:.1f}s", flush=True)
    # the reference's float path (ssl::gsvd), its own solver
    r_all = R.correlation(w.x[: t - 1 + nb], t)
    sig_f = [R.gsvd(w.k, r_all[b], path=0, threads=os.cpu_count())["sigma"] for b in range(nb)]
    print(f"float reference path: {time.time() - t0:.1f}s", flush=True)

    bins = w.bins
    cmp = {"engine_vs_fp64": [0, 0], "float_vs_fp64": [0, 0], "engine_vs_float": [0, 0]}
    zdiff = {k: 0 for k in cmp}
    hist_z, hist_groups = {}, {}
    worst_p = 0.0
    peaks_same = 0
    for b in range(nb):
        for k in range(bins):
            se, sd, sf = structure(sig[b][k]), structure(want["sigma"][b][k]), structure(sig_f[b][k])
            for name, (a, c) in (("engine_vs_fp64", (se, sd)), ("float_vs_fp64", (sf, sd)),
                                 ("engine_vs_float", (se, sf))):
                cmp[name][0] += a != c
                cmp[name][1] += 1
                zdiff[name] += a[0] != c[0]
            hist_z[sd[0]] = hist_z.get(sd[0], 0) + 1
            for gsz in sd[1]:
                if gsz > 1:
                    hist_groups[gsz] = hist_groups.get(gsz, 0) + 1
        rel = float(np.max(np.abs(pw[b] - want["power"][b]) / np.abs(want["power"][b])))
        worst_p = max(worst_p, rel)
        peaks_same += bool(np.array_equal(idx[b], want["idx"][b]))
    report = {
        "scene": "C3: reference generators (synthesize_scene + capture_noise_model over 2 s), 60-ch circular "
                 "r=0.3 m, 257 bins, 72 azimuths, targets 40/150 deg under 4 rotor noise sources, diffuse -20 dB, "
                 "T=50",
        "blocks": nb, "bins_per_block": bins, "solves": nb * bins,
        "structure": "z = #values <= 1e-5 sigma_max; tie groups = runs of kept values with gaps <= 1e-5 sigma_max "
                     "(gsvd.cpp:475-497)",
        "flip_rate": {k: {"differing_solves": v[0], "rate": v[0] / v[1], "z_differs": zdiff[k]}
                      for k, v in cmp.items()},
        "fp64_z_histogram": {str(k): v for k, v in sorted(hist_z.items())},
        "fp64_tied_group_sizes": {str(k): v for k, v in sorted(hist_groups.items())},
        "engine_vs_fp64_pbar_max_rel_err": worst_p,
        "engine_vs_fp64_identical_peaks_fraction": peaks_same / nb,
        "refine_leading": 0,
        "seconds": time.time() - t0,
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(report, f, indent=1)
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
