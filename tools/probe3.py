"""Solver phase breakdown (SSLG_PHASE_CLOCKS) for the C3 workload."""
import ctypes as C, os, sys
os.environ["SSLG_PHASE_CLOCKS"] = "1"
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl, synth, _capi
w = synth.make("c3", frames=130)
names = ["whiten", "qr", "sweeps", "sigma+backmul", "complete", "groups+phase", "store", "vanish"]
for pre in (False, True):
    eng = ssl.Engine(60, 257, window_frames=50, music=ssl.MusicConfig(num_sources=2),
                     solver=ssl.SolverConfig(precondition=pre), max_batch=32)
    eng.set_noise_model(w.k); eng.set_steering(w.h, w.dirs)
    eng.push(w.x[:50])
    out = np.zeros(8)
    _capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
    o = eng.push(w.x[50:82]); ms = eng.stage_ms()
    res = eng.read_results(32)
    _capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))
    tot = out[:8].sum(); nb = 32 * 257
    print(f"pre={pre}: jacobi {ms[1]:.2f} ms/32 blocks, sweeps {res['sweeps'].mean():.2f}; per-CTA kcycles: " +
          ", ".join(f"{n} {out[i]/nb/1e3:.1f}" for i, n in enumerate(names)) + f"; total {tot/nb/1e3:.1f}", flush=True)
    eng.close()
