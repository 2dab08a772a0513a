"""Which C3 bins fall through to canonical_kernel (worklist), and why:
per-scene histogram of the vanishing-block size z and the largest group."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import ssl, synth


def scene(kind):
    if kind == "frames":
        w = synth.make("c3", frames=130)
        w.x = w.x[:130]
        return w, w.x
    w = synth.make_pcm("c3", duration_s=(200 * 160 + 512) / 16000.0, seed=11)
    e = ssl.Engine(60, 257, max_batch=32)
    e.set_stft(ssl.StftConfig(w.frame_length, w.shift, "hann", w.bin_min, w.bin_max))
    x = e.stft(w.pcm); e.close()
    return w, x


T = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for kind in ("pcm", "frames"):
    w, x = scene(kind)
    eng = ssl.Engine(60, 257, window_frames=T, music=ssl.MusicConfig(num_sources=2), max_batch=32)
    eng.set_noise_model(w.k); eng.set_steering(w.h, w.dirs)
    # sequential frames (a repeated push would duplicate frames in the window
    # and halve R's rank)
    eng.push(x[:T]); eng.push(x[T:T + 32]); eng.synchronize()
    eng.push(x[T + 32:T + 64]); ms = eng.stage_ms()
    res = eng.read_results(32, sigma=True)
    sg = res["sigma"].reshape(-1, 60)
    conv = res["conv"].reshape(-1)
    gap = 1e-5 * sg[:, 0]
    z = (sg <= gap[:, None]).sum(1)
    dmax = []
    tied = []
    for b in range(sg.shape[0]):
        lead = 60 - z[b]; d = z[b]; i = 0
        while i < lead:
            e = i
            while e + 1 < lead and sg[b, e] - sg[b, e + 1] <= gap[b]: e += 1
            d = max(d, e - i + 1)
            if e > i: tied.append(e - i + 1)
            i = e + 1
        dmax.append(d)
    print("  tied groups per block %.2f, sizes" % (len(tied) / sg.shape[0]),
          dict(zip(*[a.tolist() for a in np.unique(tied, return_counts=True)])) if tied else {})
    dmax = np.array(dmax)
    print(kind, "stage ms", np.round(ms, 3), "blocks", sg.shape[0])
    print("  z hist", dict(zip(*[a.tolist() for a in np.unique(z, return_counts=True)])))
    print("  dmax>24", int((dmax > 24).sum()), "not conv", int((conv == 0).sum()),
          "per-bin fallthrough", np.nonzero(((dmax > 24) | (conv == 0)).reshape(32, 257).any(0))[0].tolist()[:40])
    eng.close()
