"""Solver probes (development aids, not tests; GPU required).

  python tools/solver_probes.py phases [c1|c2|c3]   per-CTA SM clocks per solver phase (SSLG_PHASE_CLOCKS;
                                                    the fused CTA solver), C3 with and without the QR
                                                    preconditioning
  python tools/solver_probes.py alone               the same clocks for ONE CTA alone (1 bin, 1 block):
                                                    the per-phase critical path without SM contention
  python tools/solver_probes.py worklist [T]        which C3 bins fall through to canonical_kernel and
                                                    why: the vanishing-block size z, tied groups, the
                                                    largest group, non-converged bins (PCM and frame scenes)

The numbers quoted in DESIGN.md section 5 ("Per-CTA phase clocks") come from
`phases c3`.
"""
import os
import sys

os.environ["SSLG_PHASE_CLOCKS"] = "1"  # read when the library creates a context
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03373_b200 import _capi, ssl, synth  # noqa: E402

PHASES = ["whiten", "qr", "sweeps", "sigma+backmul", "complete", "groups+phase", "store", "vanish"]


def _clocks(eng, out):
    _capi.check(eng.L.sslg_debug_phase_clocks(eng.h, _capi.f64p(out), 1))


def phases(cfg="c3"):
    w = synth.make(cfg, frames=130)
    m, bins = w.x.shape[1], w.x.shape[2]
    for pre in ((False, True) if m == 60 else (True,)):
        eng = ssl.Engine(m, bins, window_frames=50, music=ssl.MusicConfig(num_sources=w.ns),
                         solver=ssl.SolverConfig(precondition=pre), max_batch=32)
        eng.set_noise_model(w.k)
        eng.set_steering(w.h, w.dirs)
        eng.push(w.x[:50])
        out = np.zeros(8)
        _clocks(eng, out)  # reset
        eng.push(w.x[50:82])
        ms = eng.stage_ms()
        res = eng.read_results(32)
        _clocks(eng, out)
        nb = 32 * bins
        print(f"{cfg} m={m} precondition={pre}: stage ms {np.round(ms, 3)}, sweeps {res['sweeps'].mean():.2f}; "
              "per-CTA kcycles: " + ", ".join(f"{n} {out[i] / nb / 1e3:.1f}" for i, n in enumerate(PHASES)) +
              f"; total {out.sum() / nb / 1e3:.1f}", flush=True)
        eng.close()


def alone():
    w = synth.make("c3", frames=60)
    for b in (60, 128):
        eng = ssl.Engine(60, 1, window_frames=50, music=ssl.MusicConfig(num_sources=2), max_batch=1)
        eng.set_noise_model(w.k[b:b + 1])
        eng.set_steering(np.ascontiguousarray(w.h[:, b:b + 1]), w.dirs)
        eng.push(np.ascontiguousarray(w.x[:49, :, b:b + 1]))
        out = np.zeros(8)
        _clocks(eng, out)
        eng.push(np.ascontiguousarray(w.x[49:50, :, b:b + 1]))  # warm
        _clocks(eng, out)
        eng.push(np.ascontiguousarray(w.x[50:51, :, b:b + 1]))
        _clocks(eng, out)
        res = eng.read_results(1, sigma=True)
        print(f"bin {b} alone: sweeps {res['sweeps'].mean():.0f}; kcycles: " +
              ", ".join(f"{n} {out[i] / 1e3:.1f}" for i, n in enumerate(PHASES)) +
              f"; total {out[:8].sum() / 1e3:.1f}", flush=True)
        eng.close()


def _scene(kind):
    if kind == "frames":
        w = synth.make("c3", frames=130)
        return w, w.x[:130]
    w = synth.make_pcm("c3", duration_s=(200 * 160 + 512) / 16000.0, seed=11)
    e = ssl.Engine(60, 257, max_batch=32)
    e.set_stft(ssl.StftConfig(w.frame_length, w.shift, "hann", w.bin_min, w.bin_max))
    x = e.stft(w.pcm)
    e.close()
    return w, x


def worklist(t=50):
    for kind in ("pcm", "frames"):
        w, x = _scene(kind)
        eng = ssl.Engine(60, 257, window_frames=t, music=ssl.MusicConfig(num_sources=2), max_batch=32)
        eng.set_noise_model(w.k)
        eng.set_steering(w.h, w.dirs)
        # sequential frames (a repeated push would duplicate frames in the
        # window and halve R's rank)
        eng.push(x[:t])
        eng.push(x[t:t + 32])
        eng.synchronize()
        eng.push(x[t + 32:t + 64])
        ms = eng.stage_ms()
        res = eng.read_results(32, sigma=True)
        sg = res["sigma"].reshape(-1, 60)
        conv = res["conv"].reshape(-1)
        gap = 1e-5 * sg[:, 0]
        z = (sg <= gap[:, None]).sum(1)
        dmax, tied = [], []
        for b in range(sg.shape[0]):
            lead, d, i = 60 - z[b], z[b], 0
            while i < lead:
                e = i
                while e + 1 < lead and sg[b, e] - sg[b, e + 1] <= gap[b]:
                    e += 1
                d = max(d, e - i + 1)
                if e > i:
                    tied.append(e - i + 1)
                i = e + 1
            dmax.append(d)
        dmax = np.array(dmax)
        print(kind, "stage ms", np.round(ms, 3), "blocks", sg.shape[0])
        print("  tied groups per block %.2f" % (len(tied) / sg.shape[0]),
              dict(zip(*[a.tolist() for a in np.unique(tied, return_counts=True)])) if tied else {})
        print("  z hist", dict(zip(*[a.tolist() for a in np.unique(z, return_counts=True)])))
        print("  dmax>24", int((dmax > 24).sum()), "not conv", int((conv == 0).sum()), "per-bin fallthrough",
              np.nonzero(((dmax > 24) | (conv == 0)).reshape(32, 257).any(0))[0].tolist()[:40], flush=True)
        eng.close()


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "phases"
    rest = sys.argv[2:]
    if cmd == "phases":
        phases(*rest)
    elif cmd == "alone":
        alone()
    elif cmd == "worklist":
        worklist(*(int(v) for v in rest))
    else:
        sys.exit(__doc__)
