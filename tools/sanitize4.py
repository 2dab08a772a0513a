"""Streaming paths under compute-sanitizer (development aid): device STFT,
sample pushes across calls, asynchronous pushes with the result ring, and
the non-finite gate."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl, synth
from paper_2504_03373_b200.errors import ValidationError

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = np.load(os.path.join(root, "tests", "golden", "stft.npz"))
fl, sh, win, b0, b1 = (int(v) for v in g["hann_band_cfg"])
stft = ssl.StftConfig(fl, sh, "hann", b0, b1)
audio = g["hann_band_audio"]
m = audio.shape[0]
eng = ssl.Engine(m, stft.bin_count(), window_frames=6, music=ssl.MusicConfig(num_sources=2), max_batch=8)
rng = np.random.default_rng(1)
a = rng.standard_normal((stft.bin_count(), m, m)) + 1j * rng.standard_normal((stft.bin_count(), m, m))
eng.set_noise_model((a @ a.conj().transpose(0, 2, 1) / m + np.eye(m)).astype(np.complex64))
dirs = synth.azimuth_grid(5.0)
eng.set_steering(synth.steering(synth.circular(m, 0.05), dirs, stft.bin_min, stft.bin_max, stft.frame_length), dirs)
eng.set_stft(stft)
o = eng.push_samples(audio[:, :1500], want_power=True)
o2 = eng.push_samples(audio[:, 1500:], want_power=True)
print("sync blocks", o["n"] + o2["n"])
eng.reset_window()
tickets = [eng.push_samples_async(audio[:, s:s + 700]) for s in range(0, audio.shape[1], 700)]
print("async blocks", eng.wait_results(tickets[-1])["n"])
eng.reset_window()
bad = audio.copy()
bad[1, 2500] = np.nan
t1 = eng.push_samples_async(bad[:, :2000])
t2 = eng.push_samples_async(bad[:, 2000:])
eng.wait_results(t1)
try:
    eng.wait_results(t2)
    print("gate FAILED")
except ValidationError:
    print("gate ok")
eng.close()
