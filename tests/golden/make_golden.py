"""Generates the golden fixtures under tests/golden/ from the UNMODIFIED
reference, compiled from /root/reference/proj/src into oracle/_ref by
oracle/Makefile.  Inputs come from the reference's own seeded generators
(synthesize_scene / stft_stream / capture_noise_model / random_noise_model /
make_steering, proj/src/synth.cpp, bench.cpp); outputs from its public API
(CorrelationWindow, gsvd_reference, gsvd, calc_average_power, peak_search,
DirectionTopology::build).

Run:  python tests/golden/make_golden.py      (needs /root/reference or a
prebuilt oracle/_ref/libsslref.so)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from oracle import MusicCfg, Scene, Source  # noqa: E402


def scene_fixture(name, scene: Scene, t: int, ns: int, frames: int):
    R = oracle.ref()
    w = R.workload(scene)
    x = w.x[:frames]
    mc = MusicCfg.make(num_sources=ns)
    r = R.correlation(x, t)
    dbl = R.locate_frames(oracle.Workload(x, w.k, w.h, w.dirs), t, mc, path=2, threads=4, keep_bins=True)
    flt = R.locate_frames(oracle.Workload(x, w.k, w.h, w.dirs), t, mc, path=0, threads=4, keep_bins=True)
    g = R.gsvd(w.k, r[0], path=1, threads=4)
    gf = R.gsvd(w.k, r[0], path=0, threads=4)
    off, nbr = R.topology(w.dirs, 10.0)
    kinv = np.stack([R.mat_inverse(w.k[b], precision=1, bin_label=b) for b in range(w.bins)])
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"),
        x=x, k=w.k, h=w.h, dirs=w.dirs, t=t, ns=ns, r=r, kinv=kinv,
        sigma0=g["sigma"], e0=g["e"], sweeps0=g["iters"],
        sigma0_f=gf["sigma"], e0_f=gf["e"],
        power=dbl["power"], bin_power=dbl["bin_power"], idx=dbl["idx"], pw=dbl["pw"], low=dbl["low"],
        count=dbl["count"],
        power_f=flt["power"], bin_power_f=flt["bin_power"], idx_f=flt["idx"], count_f=flt["count"],
        topo_off=off, topo_nbr=nbr,
    )
    print(name, "frames", x.shape, "blocks", dbl["power"].shape[0], "peaks", dbl["idx"][:3].tolist())


def kat_fixture():
    """Small matrices through jacobi_svd / gsvd_reference_matrix / mat_inverse
    / hermitian_eigenvalues (gsvd.cpp:21-62, 622-716; eig.cpp:11-84)."""
    R = oracle.ref()
    rng = np.random.default_rng(2025)
    out = {}
    for n in (1, 2, 3, 5, 8, 16):
        a = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).astype(np.complex128)
        j = R.jacobi_svd(a)
        out[f"jac_a_{n}"] = a
        out[f"jac_s_{n}"] = j["sigma"]
        out[f"jac_u_{n}"] = j["u"]
        out[f"jac_vh_{n}"] = j["vh"]
        g = R.gsvd_matrix(np.eye(n), a, precision=2)
        out[f"ref_s_{n}"] = g["sigma"]
        out[f"ref_e_{n}"] = g["e"]
        # exact low-rank input (both canonicalization branches)
        if n >= 3:
            u = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
            v = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
            lr = (u @ v.conj().T).astype(np.complex64).astype(np.complex128)
            g2 = R.gsvd_matrix(np.eye(n), lr, precision=2)
            out[f"lr_a_{n}"] = lr
            out[f"lr_s_{n}"] = g2["sigma"]
            out[f"lr_e_{n}"] = g2["e"]
        k = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        k = (k @ k.conj().T / n + 0.5 * np.eye(n)).astype(np.complex64)
        k = np.triu(k) + np.triu(k, 1).conj().T
        out[f"inv_k_{n}"] = k
        out[f"inv_d_{n}"] = R.mat_inverse(k, precision=1)
        out[f"eig_{n}"] = R.hermitian_eigenvalues(k.astype(np.complex128))
    # acceptance-2 style pairs (acceptance.cpp:128-137)
    for m in (2, 4, 8, 16):
        for trial in range(3):
            kk, rr = R.random_psd_pair(m, 2, (m << 32) | trial)
            ki = R.mat_inverse(kk, precision=1)
            g = R.gsvd_matrix(ki, rr.astype(np.complex128), precision=2)
            out[f"acc_k_{m}_{trial}"] = kk
            out[f"acc_r_{m}_{trial}"] = rr
            out[f"acc_s_{m}_{trial}"] = g["sigma"]
            out[f"acc_e_{m}_{trial}"] = g["e"]
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)
    print("kat", len(out), "arrays")


def stft_fixture():
    """Audio through the reference's stft_stream (stft.cpp:38-68, fft.hpp:15-68):
    PCM from synthesize_scene, frames from the reference itself."""
    R = oracle.ref()
    out = {}
    cases = [
        ("hann_band", Scene(mics=8, radius=0.05, duration_s=0.25, seed=21, diffuse_db=-20, bin_min=16, bin_max=88,
                            sources=[Source(40), Source(150, kind="tone", freq=1000.0)])),
        ("rect_full", Scene(mics=3, radius=0.05, duration_s=0.12, seed=4, window="rectangular", bin_min=0,
                            bin_max=256, sources=[Source(10), Source(200, kind="tone", freq=2500.0)])),
        ("hann_256", Scene(mics=5, radius=0.05, duration_s=0.1, seed=8, frame_length=256, shift=100, bin_min=3,
                           bin_max=128, diffuse_db=-10, sources=[Source(300)])),
        # non-power-of-two lengths: real_dft_half's direct sum (fft.hpp:55-65)
        ("hann_480", Scene(mics=4, radius=0.05, duration_s=0.12, seed=12, frame_length=480, shift=160, bin_min=10,
                           bin_max=90, diffuse_db=-20, sources=[Source(60)])),
        ("rect_300", Scene(mics=3, radius=0.05, duration_s=0.08, seed=13, window="rectangular", frame_length=300,
                           shift=100, bin_min=0, bin_max=150, sources=[Source(120, kind="tone", freq=900.0)])),
    ]
    for name, sc in cases:
        w = R.workload(sc, with_audio=True)
        out[f"{name}_audio"] = w.audio
        out[f"{name}_frames"] = w.x
        out[f"{name}_cfg"] = np.array([sc.frame_length, sc.shift, 0 if sc.window == "hann" else 1, sc.bin_min,
                                       sc.bin_max], np.int64)
        print("stft", name, w.audio.shape, "->", w.x.shape)
    np.savez_compressed(os.path.join(HERE, "stft.npz"), **out)


def main():
    if "--stft" in sys.argv:
        stft_fixture()
        return
    # C1 shape, reduced band: 8-ch circular, 2 white sources + diffuse, captured K
    scene_fixture("c1_band", Scene(mics=8, radius=0.05, duration_s=0.5, seed=7, diffuse_db=-20, bin_min=16,
                                   bin_max=48, sources=[Source(40), Source(150)], noise="captured"),
                  t=10, ns=2, frames=16)
    # C2 shape, reduced band: 16-ch, random noise model
    scene_fixture("c2_band", Scene(mics=16, radius=0.05, duration_s=0.5, seed=3, diffuse_db=-25, bin_min=20,
                                   bin_max=31, sources=[Source(75), Source(200, level_db=-3)], noise="random",
                                   noise_seed=5),
                  t=20, ns=2, frames=24)
    # identity noise (SEVD-MUSIC special case), tone + white, rank-deficient T < m
    scene_fixture("c1_identity_lowrank", Scene(mics=12, radius=0.06, duration_s=0.4, seed=9, bin_min=10,
                                               bin_max=25, sources=[Source(100, kind="tone", freq=700.0),
                                                                    Source(250)], noise="identity"),
                  t=6, ns=2, frames=10)
    kat_fixture()
    stft_fixture()


if __name__ == "__main__":
    main()
