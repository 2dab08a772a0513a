"""60-channel engine run for compute-sanitizer (development aid): the
flagship kernels on a few bins, a short window (big_vanish) and the DMMA
spectrum with its bulk-copy staging."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl, synth
w = synth.make("c3", frames=40)
sl = slice(100, 104)
for t in (24, 30):
    eng = ssl.Engine(60, 4, window_frames=t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=4)
    eng.set_noise_model(np.ascontiguousarray(w.k[sl]))
    eng.set_steering(np.ascontiguousarray(w.h[:, sl]), w.dirs)
    out = eng.push(np.ascontiguousarray(w.x[:t + 2, :, sl]), want_power=True)
    print("T", t, "blocks", out["n"], "idx", out["idx"].tolist())
    eng.close()
