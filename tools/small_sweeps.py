import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2504_03373_b200 import ssl, synth
for cfg in ("c1", "c2"):
    w = synth.make(cfg, frames=60)
    eng = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=16)
    eng.set_noise_model(w.k); eng.set_steering(w.h, w.dirs)
    eng.push(w.x[:w.t-1]); o = eng.push(w.x[w.t-1:w.t+7]); r = eng.read_results(o["n"], sigma=True)
    print(cfg, os.environ.get("SSLG_SMALL_CTA","0"), "sweeps mean", r["sweeps"].mean(), "max", r["sweeps"].max(), "conv", r["conv"].mean())
