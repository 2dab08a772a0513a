"""GPU STFT front end: SampleBlock -> SpectrumFrame on the
device, bit-identical to the reference's stft_stream (stft.cpp:38-68,
fft.hpp:15-68; frames in tests/golden/stft.npz were produced by the compiled
reference from the same PCM), and the sample-driven run_locate
(pipeline.cpp:210-247) agreeing exactly with the frame-driven path.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "stft.npz")
CASES = ["hann_band", "rect_full", "hann_256", "hann_480", "rect_300"]


def _cfg(g, name):
    from paper_2504_03373_b200 import ssl

    fl, sh, win, b0, b1 = (int(v) for v in g[name + "_cfg"])
    return ssl.StftConfig(fl, sh, "hann" if win == 0 else "rectangular", b0, b1)


def _engine(m, stft, t=6, ns=2, max_batch=8, seed=3):
    from paper_2504_03373_b200 import ssl, synth

    eng = ssl.Engine(m, stft.bin_count(), window_frames=t, music=ssl.MusicConfig(num_sources=ns),
                     max_batch=max_batch)
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((stft.bin_count(), m, m)) + 1j * rng.standard_normal((stft.bin_count(), m, m))
    k = (a @ a.conj().transpose(0, 2, 1) / m + np.eye(m)).astype(np.complex64)
    eng.set_noise_model(k)
    mics = synth.circular(m, 0.05)
    dirs = synth.azimuth_grid(5.0)
    eng.set_steering(synth.steering(mics, dirs, stft.bin_min, stft.bin_max, stft.frame_length), dirs)
    eng.set_stft(stft)
    return eng


@pytest.mark.parametrize("name", CASES)
def test_device_stft_bit_exact(name):
    from paper_2504_03373_b200 import ssl

    g = np.load(GOLDEN)
    stft = _cfg(g, name)
    audio = g[name + "_audio"]
    eng = ssl.Engine(audio.shape[0], stft.bin_count(), max_batch=4)  # several chunks
    eng.set_stft(stft)
    out = eng.stft(audio)
    want = g[name + "_frames"]
    assert out.shape == want.shape
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    eng.close()


def test_push_samples_matches_push_frames_in_any_chunking():
    g = np.load(GOLDEN)
    stft = _cfg(g, "hann_band")
    audio = g["hann_band_audio"]
    frames = g["hann_band_frames"]
    ref = _engine(audio.shape[0], stft)
    want = ref.push(frames, want_power=True)
    ref.close()
    for cuts in ([audio.shape[1]], [1000, 1, 511, 2488], [160] * 25):
        eng = _engine(audio.shape[0], stft)
        got = dict(n=0, idx=[], power=[], frame_index=[])
        pos = 0
        for c in cuts:
            c = min(c, audio.shape[1] - pos)
            o = eng.push_samples(audio[:, pos:pos + c], want_power=True)
            pos += c
            got["n"] += o["n"]
            got["idx"] += list(o["idx"])
            got["power"] += list(o["power"])
            got["frame_index"] += list(o["frame_index"])
        eng.close()
        assert got["n"] == want["n"]
        assert np.array_equal(np.array(got["frame_index"]), want["frame_index"])
        assert np.array_equal(np.array(got["idx"]), want["idx"])
        assert np.array_equal(np.array(got["power"]), want["power"])


def test_run_locate_on_samples_matches_frames():
    from paper_2504_03373_b200 import ssl, synth

    g = np.load(GOLDEN)
    stft = _cfg(g, "hann_band")
    audio = g["hann_band_audio"]
    m = audio.shape[0]
    rng = np.random.default_rng(1)
    a = rng.standard_normal((stft.bin_count(), m, m)) + 1j * rng.standard_normal((stft.bin_count(), m, m))
    k = (a @ a.conj().transpose(0, 2, 1) / m + np.eye(m)).astype(np.complex64)
    dirs = synth.azimuth_grid(5.0)
    h = synth.steering(synth.circular(m, 0.05), dirs, stft.bin_min, stft.bin_max, stft.frame_length)
    noise = ssl.NoiseModel(ssl.CorrelationSet(m, k))
    steering = ssl.SteeringField(m, stft.bin_min, stft.bin_max, dirs, h)
    music = ssl.MusicConfig(num_sources=2)
    a_out, b_out = [], []
    na = ssl.run_locate_samples(audio, stft, 6, noise, steering, music=music, sink=a_out.append)
    nb = ssl.run_locate(g["hann_band_frames"], 6, noise, steering, music=music, sink=b_out.append)
    assert na == nb == len(a_out) > 0
    for fa, fb in zip(a_out, b_out):
        assert fa.frame_index == fb.frame_index
        assert [e.direction_index for e in fa.estimates] == [e.direction_index for e in fb.estimates]
        assert [e.power for e in fa.estimates] == [e.power for e in fb.estimates]


def test_stft_validation():
    from paper_2504_03373_b200 import ssl
    from paper_2504_03373_b200.errors import ValidationError

    eng = ssl.Engine(2, 73)
    with pytest.raises(ValidationError):
        eng.set_stft(ssl.StftConfig(512, 160, "hann", 16, 90))  # band != engine bins
    eng.set_stft(ssl.StftConfig(480, 160, "hann", 16, 88))  # other lengths: the direct sum (fft.hpp:55-65)
    with pytest.raises(ValidationError):
        eng.set_stft(ssl.StftConfig(5000, 160, "hann", 16, 88))  # direct sum capped at 4096 on the device
    with pytest.raises(ValidationError):
        eng.set_stft(ssl.StftConfig(512, 600, "hann", 16, 88))  # shift > frame_length
    eng.set_stft(ssl.StftConfig())
    assert eng.stft(np.zeros((2, 400), np.float32)).shape == (0, 2, 73)
    eng.close()


def test_non_finite_samples_rejected_window_unchanged():
    """A non-finite sample makes its frames non-finite: the push fails with the
    reference's message (instantaneous_correlation, correlation.cpp:16-17),
    the correlation window keeps its state, and a reset recovers the stream."""
    from paper_2504_03373_b200.errors import ValidationError

    g = np.load(GOLDEN)
    stft = _cfg(g, "hann_band")
    audio = g["hann_band_audio"].copy()
    frames = g["hann_band_frames"]
    eng = _engine(audio.shape[0], stft)
    first = eng.push_samples(audio[:, :2000], want_power=True)
    bad = audio[:, 2000:2400].copy()
    bad[1, 37] = np.nan
    with pytest.raises(ValidationError, match="non-finite"):
        eng.push_samples(bad)
    eng.reset_window()
    again = eng.push_samples(audio, want_power=True)
    ref = _engine(audio.shape[0], stft)
    want = ref.push(frames, want_power=True)
    assert np.array_equal(again["power"], want["power"])
    assert first["n"] <= want["n"]
    eng.close()
    ref.close()


def test_async_pushes_match_the_synchronous_stream():
    """sslg_push_samples_async / sslg_wait_results: many
    pushes in flight, collected later, give exactly the synchronous results;
    a non-finite value stops the stream on the device and reports the
    reference's error; a reset restarts it."""
    from paper_2504_03373_b200.errors import ValidationError

    g = np.load(GOLDEN)
    stft = _cfg(g, "hann_band")
    audio = g["hann_band_audio"]
    frames = g["hann_band_frames"]
    ref = _engine(audio.shape[0], stft)
    want = ref.push(frames, want_power=True)
    ref.close()
    eng = _engine(audio.shape[0], stft)
    eng.set_async_power(True)
    tickets = [eng.push_samples_async(audio[:, a:a + 700]) for a in range(0, audio.shape[1], 700)]
    got = eng.wait_results(tickets[-1], want_power=True)
    assert got["n"] == want["n"]
    assert np.array_equal(got["frame_index"], want["frame_index"])
    assert np.array_equal(got["power"], want["power"])
    for b in range(got["n"]):
        c = int(got["count"][b])
        assert np.array_equal(got["idx"][b][:c], want["idx"][b][:c])
    # poison: NaN in the second half
    eng.reset_window()
    bad = audio.copy()
    bad[2, 2500] = np.inf
    t1 = eng.push_samples_async(bad[:, :2000])
    t2 = eng.push_samples_async(bad[:, 2000:])
    ok = eng.wait_results(t1)
    assert ok["n"] > 0
    with pytest.raises(ValidationError, match="non-finite"):
        eng.wait_results(t2)
    with pytest.raises(ValidationError):
        eng.push_samples(audio[:, :1000])
    eng.reset_window()
    again = eng.push_samples(audio, want_power=True)
    assert np.array_equal(again["power"], want["power"])
    eng.close()
