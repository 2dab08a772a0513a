"""Solver phase latency of ONE CTA alone (1 bin, 1 block) vs the full C3
batch: separates the per-phase critical path from SM contention."""
import os, sys
os.environ["SSLG_PHASE_CLOCKS"] = "1"
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl, synth, _capi
w = synth.make("c3", frames=60)
names = ["whiten", "qr", "sweeps", "sigma+backmul", "complete", "groups+phase", "store", "vanish"]
for b in (60, 128):
    eng = ssl.Engine(60, 1, window_frames=50, music=ssl.MusicConfig(num_sources=2), max_batch=1)
    eng.set_noise_model(w.k[b:b + 1]); eng.set_steering(np.ascontiguousarray(w.h[:, b:b + 1]), w.dirs)
    eng.push(np.ascontiguousarray(w.x[:49, :, b:b + 1]))
    out = np.zeros(8)
    _capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
    eng.push(np.ascontiguousarray(w.x[49:50, :, b:b + 1]))
    _capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
    eng.push(np.ascontiguousarray(w.x[50:51, :, b:b + 1]))
    _capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
    res = eng.read_results(1, sigma=True)
    print(f"bin {b} alone: sweeps {res['sweeps'].mean():.0f}; kcycles: " +
          ", ".join(f"{n} {out[i]/1e3:.1f}" for i, n in enumerate(names)) + f"; total {out[:8].sum()/1e3:.1f}", flush=True)
    eng.close()
