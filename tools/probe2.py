"""Parity + timing of refine_leading on/off (development aid)."""
import os, sys, time, functools
print = functools.partial(print, flush=True)  # noqa: A001
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2504_03373_b200 import ssl, synth

P = oracle.port()
for name in ["c1_band", "c2_band", "c1_identity_lowrank"]:
    g = dict(np.load(f"tests/golden/{name}.npz"))
    t, ns = int(g["t"]), int(g["ns"])
    for refine, pre in ((False, False), (False, True), (True, True)):
        eng = ssl.Engine(g["x"].shape[1], g["x"].shape[2], window_frames=t, music=ssl.MusicConfig(num_sources=ns),
                         solver=ssl.SolverConfig(refine_leading=refine, precondition=pre), max_batch=32)
        eng.set_noise_model(g["k"]); eng.set_steering(g["h"], g["dirs"])
        out = eng.push(g["x"], want_power=True); n = out["n"]
        res = eng.read_results(n, power=True, bin_power=True, sigma=True)
        sig, e, _, _ = eng.gsvd(g["r"][0])
        bp = max(np.max(np.abs(res["bin_power"][b] - g["bin_power"][b]) / g["bin_power"][b]) for b in range(n))
        pb = max(np.max(np.abs(res["power"][b] - g["power"][b]) / g["power"][b]) for b in range(n))
        pk = all(np.array_equal(out["idx"][b][:out["count"][b]], g["idx"][b][:g["count"][b]]) for b in range(n))
        print(f"{name} refine={refine} pre={pre}: E0 maxabs {np.max(np.abs(e[0]-g['e0'])):.2e} sigma {np.max(np.abs(sig[0]-g['sigma0'])/g['sigma0'][:, :1]):.2e} binP {bp:.2e} Pbar {pb:.2e} peaks {pk}")
        eng.close()

w = synth.make("c3", frames=90)
r = P.correlation(w.x[:52], 50)
ref = P.locate(w.x[:52], w.k, w.h, w.dirs, 50, 2, keep_bins=True)
for refine, pre in ((False, False), (False, True), (True, True)):
    eng = ssl.Engine(60, 257, window_frames=50, music=ssl.MusicConfig(num_sources=2),
                     solver=ssl.SolverConfig(refine_leading=refine, precondition=pre), max_batch=64)
    eng.set_noise_model(w.k); eng.set_steering(w.h, w.dirs)
    out = eng.push(w.x[:52], want_power=True); n = out["n"]
    res = eng.read_results(n, power=True, bin_power=True, sigma=True)
    bp = max(np.max(np.abs(res["bin_power"][b] - ref["bin_power"][b]) / ref["bin_power"][b]) for b in range(n))
    pb = max(np.max(np.abs(res["power"][b] - ref["power"][b]) / ref["power"][b]) for b in range(n))
    sg = max(np.max(np.abs(res["sigma"][b] - ref["sigma"][b]) / ref["sigma"][b][:, :1]) for b in range(n))
    pk = all(np.array_equal(out["idx"][b][:out["count"][b]], ref["idx"][b]) for b in range(n))
    print(f"C3 refine={refine} pre={pre}: sigma {sg:.2e} binP {bp:.2e} Pbar {pb:.2e} peaks {pk} idx {out['idx'][:3].tolist()} sweeps {res['sweeps'].mean():.1f}")
    x = w.x[52:52+32]
    o = eng.push(x); ms = eng.stage_ms()
    print(f"C3 refine={refine} pre={pre}: push32 stage_ms {ms} -> {1e3*(ms[1]+ms[2])/32:.0f} us/block gsvd")
    eng.close()
