"""Solver phase breakdown (SSLG_PHASE_CLOCKS) for a small-array config (c1/c2)."""
import os, sys
os.environ["SSLG_PHASE_CLOCKS"] = "1"
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl, synth, _capi
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = synth.make(cfg, frames=130)
m, bins = w.x.shape[1], w.x.shape[2]
names = ["whiten", "qr", "sweeps", "sigma+backmul", "complete", "groups+phase", "store", "vanish"]
eng = ssl.Engine(m, bins, window_frames=50, music=ssl.MusicConfig(num_sources=w.ns), max_batch=32)
eng.set_noise_model(w.k); eng.set_steering(w.h, w.dirs)
eng.push(w.x[:50])
out = np.zeros(8)
_capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
eng.push(w.x[50:82]); ms = eng.stage_ms()
res = eng.read_results(32)
_capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
nb = 32 * bins
print(f"{cfg} m={m}: stage ms {np.round(ms, 3)}, sweeps {res['sweeps'].mean():.2f}; per-CTA kcycles: " +
      ", ".join(f"{n} {out[i]/nb/1e3:.1f}" for i, n in enumerate(names)) + f"; total {out.sum()/nb/1e3:.1f}")
