"""Small engine run for compute-sanitizer (development aid)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl
g = dict(np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/c1_band.npz")))
t, ns = int(g["t"]), int(g["ns"])
m, bins = g["x"].shape[1], g["x"].shape[2]
eng = ssl.Engine(m, bins, window_frames=t, music=ssl.MusicConfig(num_sources=ns), max_batch=16)
eng.set_noise_model(g["k"])
eng.set_steering(g["h"], g["dirs"])
out = eng.push(g["x"], want_power=True)
print("blocks", out["n"], "idx", out["idx"].tolist(), "ref", g["idx"].tolist())
print("power rel", np.max(np.abs(out["power"] - g["power"]) / g["power"]))
