"""Development aid: mean Jacobi sweeps per bin and the sweep phase's SM clocks
per bin on a C3 scene, for A/B comparisons of sweep orderings
(SSLG_BLOCK_SWEEPS=0/1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SSLG_PHASE_CLOCKS", "1")
from paper_2504_03373_b200 import _capi, ssl, synth  # noqa: E402
import ctypes as C  # noqa: E402

w = synth.make("c3", frames=90)
eng = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=32)
eng.set_noise_model(w.k)
eng.set_steering(w.h, w.dirs)
eng.push(w.x[: w.t - 1])
clk = np.zeros(8)
L = _capi.load()
L.sslg_debug_phase_clocks(eng.h, clk.ctypes.data_as(C.POINTER(C.c_double)), 1)
eng.push(w.x[w.t - 1: w.t - 1 + 32])
L.sslg_debug_phase_clocks(eng.h, clk.ctypes.data_as(C.POINTER(C.c_double)), 1)
r = eng.read_results(32, sigma=True)
nb = 32 * w.bins
print(f"BS={os.environ.get('SSLG_BLOCK_SWEEPS', '0')} sweeps/bin {r['sweeps'].mean():.3f} "
      f"phase clocks per bin (kcycles): " + " ".join(f"{c / nb / 1e3:.1f}" for c in clk[:7]))
