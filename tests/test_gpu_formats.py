"""GPU: the on-disk inputs into a device context and the device noise
capture, against the compiled reference.

  capture_noise_model     K bit-identical to the reference's (synth.cpp:329-373)
                          on the same noise-only PCM, PD-gated like it
  NoiseModel::from_file   loaded K^-1 bit-identical to set_noise_model's
  load_steering           spectrum identical to the one from set_steering
  JSONL through run_locate  records field-identical to the reference's own
                          run_locate estimates formatted by nlohmann
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype in (np.complex128, np.float64) else np.uint32)


def noise_scene(mics=8, radius=0.05, duration=1.0, seed=3):
    import oracle

    src = [oracle.Source(45.0, level_db=-3.0, noise_role=True), oracle.Source(200.0, 10.0, level_db=-6.0,
                                                                             noise_role=True)]
    return oracle.Scene(mics=mics, radius=radius, duration_s=duration, seed=seed, diffuse_db=-20.0, sources=src,
                        bin_min=16, bin_max=88, noise="captured", noise_duration_s=duration)


@pytest.mark.parametrize("mics,radius", [(8, 0.05), (16, 0.05), (60, 0.3)])
def test_capture_noise_model_bit_exact(ref, mics, radius):
    """Every source plays the noise role and the capture lasts as long as the
    scene, so the reference's capture_noise_model re-synthesizes exactly the
    workload's audio: its K and ours from that PCM must agree bit for bit."""
    from paper_2504_03373_b200 import ssl

    sc = noise_scene(mics, radius)
    w = ref.workload(sc, with_audio=True)
    stft = ssl.StftConfig(512, 160, "hann", 16, 88)
    got = ssl.NoiseModel.capture(w.audio, stft)
    assert got.k.bins.shape == w.k.shape
    assert np.array_equal(bits(got.k.bins), bits(w.k))


def test_capture_installs_and_gates():
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(4)
    m = 4
    eng = ssl.Engine(m, 9, max_batch=4)
    eng.set_stft(ssl.StftConfig(512, 160, "hann", 0, 8))
    with pytest.raises(ssl.ValidationError, match="shorter than one frame"):
        eng.capture_noise_model(np.zeros((m, 300), np.float32))
    # rank-deficient noise (one channel silent): not positive definite
    pcm = rng.standard_normal((m, 8000)).astype(np.float32)
    pcm[2] = 0.0
    with pytest.raises(ssl.NumericalError, match="not positive definite"):
        eng.capture_noise_model(pcm)
    pcm[2] = rng.standard_normal(8000)
    k = eng.capture_noise_model(pcm)  # installed: the inverses are the set_noise_model ones
    ref = ssl.Engine(m, 9, max_batch=4)
    ref.set_noise_model(k)
    assert np.array_equal(bits(eng.noise_inverse(1)), bits(ref.noise_inverse(1)))
    eng.close()
    ref.close()


def test_noise_model_and_steering_from_files(golden, tmp_path):
    from paper_2504_03373_b200 import formats, ssl

    g = golden("c2_band")
    m, bins = g["k"].shape[1], g["k"].shape[0]
    kp, sp = str(tmp_path / "k.sslc"), str(tmp_path / "h.steer")
    formats.save_correlation(kp, g["k"], int(g["t"]))
    formats.save_steering(sp, ssl.SteeringField(m, 16, 16 + bins - 1, g["dirs"], g["h"]))
    a = ssl.Engine(m, bins, window_frames=int(g["t"]), music=ssl.MusicConfig(num_sources=int(g["ns"])), max_batch=32)
    assert a.load_noise_model(kp) == int(g["t"])
    assert a.load_steering(sp) == 16
    b = ssl.Engine(m, bins, window_frames=int(g["t"]), music=ssl.MusicConfig(num_sources=int(g["ns"])), max_batch=32)
    b.set_noise_model(g["k"])
    b.set_steering(g["h"], g["dirs"])
    assert np.array_equal(bits(a.noise_inverse(1)), bits(b.noise_inverse(1)))
    pa = a.push(g["x"], want_power=True)
    pb = b.push(g["x"], want_power=True)
    assert np.array_equal(pa["power"], pb["power"]) and np.array_equal(pa["idx"], pb["idx"])
    # a noise file of the wrong shape is refused
    formats.save_correlation(kp, g["k"][:3], 1)
    with pytest.raises(ssl.ValidationError, match="bin count"):
        a.load_noise_model(kp)
    a.close()
    b.close()


def test_noise_file_pd_gate(tmp_path):
    """NoiseModel::from_file gates positive definiteness (gsvd.cpp:729-734)."""
    from paper_2504_03373_b200 import formats, ssl

    k = np.zeros((3, 2, 2), np.complex64)
    k[:, 0, 0] = k[:, 1, 1] = 1.0
    k[1, 1, 1] = -1.0
    p = str(tmp_path / "bad.sslc")
    formats.save_correlation(p, k, 1)
    with pytest.raises(ssl.NumericalError, match="not positive definite at bin 1"):
        ssl.NoiseModel.from_file(p)


def test_jsonl_of_run_locate_matches_the_reference(ref, golden):
    """run_locate_to_stream's records (pipeline.cpp:268-283) from our
    estimates vs the reference's estimates formatted by nlohmann: the same
    directions, flags and keys; powers within the P-bar tolerance."""
    from paper_2504_03373_b200 import formats, ssl

    g = golden("c1_band")
    t, ns = int(g["t"]), int(g["ns"])
    m, bins = g["x"].shape[1], g["x"].shape[2]
    steer = ssl.SteeringField(m, 0, bins - 1, g["dirs"], g["h"])
    noise = ssl.NoiseModel(ssl.CorrelationSet(m, g["k"]))
    lines = []
    ssl.run_locate(g["x"], t, noise, steer, music=ssl.MusicConfig(num_sources=ns),
                   sink=lambda fe: lines.append(formats.format_estimates_json(fe.frame_index, fe.estimates,
                                                                                g["dirs"])))
    assert len(lines) == g["idx"].shape[0]
    for b, line in enumerate(lines):
        c = int(g["count"][b])
        want = json.loads(ref.format_estimates(t - 1 + b, g["idx"][b][:c], g["dirs"], g["pw"][b][:c],
                                               g["low"][b][:c].astype(np.uint8)))
        got = json.loads(line)
        assert got["frame"] == want["frame"]
        assert [list(e) for e in got["estimates"]] == [list(e) for e in want["estimates"]]
        for eg, ew in zip(got["estimates"], want["estimates"]):
            assert (eg["direction"], eg["azimuth_deg"], eg["elevation_deg"], eg["low_power"]) == \
                (ew["direction"], ew["azimuth_deg"], ew["elevation_deg"], ew["low_power"])
            assert eg["power"] == pytest.approx(ew["power"], rel=1e-8)
