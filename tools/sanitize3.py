"""Solver corner paths under compute-sanitizer (development aid): the
generic canonical kernel (refine mode, a tied group above kZMax), the
sequential vanishing picker (rejected candidates), generic m and m = 16."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl


def run(m, r, k, solver=None):
    eng = ssl.Engine(m, r.shape[0], window_frames=2, max_batch=2, solver=solver)
    eng.set_noise_model(k)
    sigma, e, _, conv = eng.gsvd(r)
    eng.close()
    return sigma, conv


rng = np.random.default_rng(3)
m, bins = 60, 2
eye = np.broadcast_to(np.eye(m, dtype=np.complex64), (bins, m, m)).copy()
# tied group of 30
s = np.concatenate([np.linspace(9.0, 5.0, 10), np.full(30, 2.0), np.linspace(1.5, 0.5, 20)])
r = np.empty((bins, m, m), np.complex64)
for b in range(bins):
    q, _ = np.linalg.qr(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))
    r[b] = (q * s) @ q.conj().T
print("tied30", run(m, r, eye)[1].all())
# rejected candidates, z = 30
x = rng.standard_normal((bins, m, 30)) + 1j * rng.standard_normal((bins, m, 30))
x[:, 0, 2:] = 0; x[:, 2, 2:] = 0; x[:, :, :2] = 0; x[:, 0, 0] = 3.0; x[:, 2, 1] = 2.0
r2 = (x @ x.conj().transpose(0, 2, 1) / 30).astype(np.complex64)
print("reject", run(m, r2, eye)[1].all())
# refine mode
print("refine", run(m, r2, eye, ssl.SolverConfig(refine_leading=True))[1].all())
# generic m = 37 and m = 16, rank deficient
for mm in (37, 16):
    xb = rng.standard_normal((bins, mm, mm // 2)) + 1j * rng.standard_normal((bins, mm, mm // 2))
    rr = (xb @ xb.conj().transpose(0, 2, 1)).astype(np.complex64)
    kk = np.broadcast_to(np.eye(mm, dtype=np.complex64), (bins, mm, mm)).copy()
    print("m", mm, run(mm, rr, kk)[1].all())
