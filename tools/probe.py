"""Quick GPU probe: parity of the engine against the CPU oracle on a small
scene and a first timing of the C3 block.  Development aid, not a test."""
import os
import sys
import time
import functools
print = functools.partial(print, flush=True)  # noqa: A001

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from oracle import MusicCfg, Scene, Source  # noqa: E402
from paper_2504_03373_b200 import ssl  # noqa: E402


def compare(tag, w, t, ns, frames=None, refine=True):
    R, P = oracle.ref(), oracle.port()
    x = w.x if frames is None else w.x[:frames]
    eng = ssl.Engine(w.m, w.bins, window_frames=t, music=ssl.MusicConfig(num_sources=ns),
                     solver=ssl.SolverConfig(refine_leading=refine), max_batch=max(1, x.shape[0] - t + 1) + t)
    eng.set_noise_model(w.k)
    eng.set_steering(w.h, w.dirs)
    t0 = time.time()
    print(f"[{tag}] pushing {x.shape}")
    out = eng.push(x, want_power=True)
    n = out["n"]
    res = eng.read_results(n, power=True, bin_power=True, sigma=True)
    print(f"[{tag}] engine push {time.time()-t0:.3f}s blocks={n} stage_ms={eng.stage_ms()} launches={eng.launch_count()}")
    print(f"[{tag}] oracle locate ...")
    t0 = time.time()
    ref = P.locate(x, w.k, w.h, w.dirs, t, ns, keep_bins=True)
    print(f"[{tag}] oracle done {time.time()-t0:.1f}s")
    sig_err = max(np.max(np.abs(res["sigma"][b] - ref["sigma"][b]) / ref["sigma"][b][:, :1]) for b in range(n))
    bp_rel = max(np.max(np.abs(res["bin_power"][b] - ref["bin_power"][b]) / np.abs(ref["bin_power"][b])) for b in range(n))
    p_rel = max(np.max(np.abs(res["power"][b] - ref["power"][b]) / np.abs(ref["power"][b])) for b in range(n))
    same = all(np.array_equal(out["idx"][b][: out["count"][b]], ref["idx"][b]) for b in range(n))
    print(f"[{tag}] sigma max rel-to-smax {sig_err:.3e}  binP max rel {bp_rel:.3e}  Pbar max rel {p_rel:.3e}  peaks identical {same}")
    print(f"[{tag}] sweeps mean {res['sweeps'].mean():.2f} max {res['sweeps'].max()} conv {res['conv'].all()}")
    return eng


def main():
    R = oracle.ref()
    # C1-like: 8 ch, 257 bins, 72 dirs, 2 white sources + diffuse, captured K
    w1 = R.workload(Scene(mics=8, radius=0.05, duration_s=0.6, seed=7, diffuse_db=-20,
                          sources=[Source(40), Source(150)], noise="captured"))
    compare("C1", w1, 50, 2, frames=54)
    # C3-like
    srcs = [Source(40, level_db=0), Source(150, level_db=0)] + \
           [Source(a, level_db=0, noise_role=True) for a in (45, 135, 225, 315)]
    t0 = time.time()
    w3 = R.workload(Scene(mics=60, geometry="circular", radius=0.3, duration_s=0.75, seed=11, diffuse_db=-20,
                          sources=srcs, noise="captured", noise_duration_s=2.0))
    print(f"C3 workload {time.time()-t0:.1f}s")
    eng = compare("C3", w3, 50, 2, frames=52)
    # timing: repeated pushes of 16 frames
    eng2 = ssl.Engine(60, 257, window_frames=50, music=ssl.MusicConfig(num_sources=2), max_batch=16)
    eng2.set_noise_model(w3.k)
    eng2.set_steering(w3.h, w3.dirs)
    eng2.push(w3.x[:50])
    for rep in range(3):
        x = w3.x[50 + (rep % 1):50 + 16 + (rep % 1)] if w3.x.shape[0] >= 66 else np.tile(w3.x[:16], (1, 1, 1))
        t0 = time.time()
        o = eng2.push(x)
        dt = time.time() - t0
        print(f"push16 wall {dt*1e3:.2f} ms blocks {o['n']} stage_ms {eng2.stage_ms()}")


if __name__ == "__main__":
    main()
