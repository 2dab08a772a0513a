"""GPU: error behaviour of the engine's streaming entry points.

* synchronous calls are refused while asynchronous pushes are uncollected;
* the device-frame push gates on the device without a host sync and reports
  a non-finite frame at the next synchronizing call, rewinding the window;
* run_locate hands the blocks before a non-finite frame to the sink before
  it raises (the reference's per-frame loop, pipeline.cpp:227-245);
* sslg_wait_results refuses a too-small result array without consuming.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def engine_for(g, **kw):
    from paper_2504_03373_b200 import ssl

    t, ns = int(g["t"]), int(g["ns"])
    m, bins = g["x"].shape[1], g["x"].shape[2]
    eng = ssl.Engine(m, bins, window_frames=t, music=ssl.MusicConfig(num_sources=ns),
                     max_batch=kw.pop("max_batch", 8), **kw)
    eng.set_noise_model(g["k"])
    eng.set_steering(g["h"], g["dirs"])
    return eng


def test_device_push_gates_on_the_device_and_rewinds(golden):
    import torch

    from paper_2504_03373_b200 import ssl

    g = golden("c1_band")
    t = int(g["t"])
    x = g["x"]
    eng = engine_for(g, max_batch=4)
    xd = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
    bad = x[t + 1: t + 3].copy()
    bad[1, 2, 3] = np.inf
    bd = torch.from_numpy(np.ascontiguousarray(bad).view(np.float32)).cuda()
    pos = 0
    while pos < t:  # fill + first emitted block
        n = min(4, t - pos)
        eng.push_device(xd[pos:pos + n].data_ptr(), n)
        pos += n
    eng.push_device(bd.data_ptr(), 2)  # returns without a host sync
    eng.push_device(xd[t + 1:t + 2].data_ptr(), 1)  # skipped on the device (stream stopped)
    with pytest.raises(ssl.ValidationError, match="non-finite"):
        eng.read_results(1)
    # the window is back to frames [0, t): continuing with frame t+1 matches a
    # clean stream that never saw the failed pushes
    n = eng.push_device(xd[t + 1:t + 2].data_ptr(), 1)
    assert n == 1
    got = eng.read_results(1, power=True)
    clean = engine_for(g, max_batch=64)
    want = clean.push(np.concatenate([x[:t], x[t + 1:t + 2]]), want_power=True)
    assert np.array_equal(got["power"][0], want["power"][-1])
    eng.close()
    clean.close()


def test_sync_calls_refused_while_async_pending():
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(1)
    m, bins = 4, 9
    eng = ssl.Engine(m, bins, window_frames=3, max_batch=4)
    eng.set_noise_identity()
    h = (rng.standard_normal((12, bins, m)) + 1j * rng.standard_normal((12, bins, m))).astype(np.complex64)
    eng.set_steering(h, np.array([[30.0 * i, 0.0] for i in range(12)]))
    eng.set_stft(ssl.StftConfig(512, 160, "hann", 0, bins - 1))
    pcm = rng.standard_normal((m, 4000)).astype(np.float32)
    tk = eng.push_samples_async(pcm[:, :2000])
    frames = (rng.standard_normal((2, m, bins)) + 0j).astype(np.complex64)
    for call in (lambda: eng.push(frames), lambda: eng.push_samples(pcm[:, :500]),
                 lambda: eng.gsvd(np.zeros((bins, m, m), np.complex64)), lambda: eng.correlation(frames),
                 lambda: eng.set_steering(h, np.array([[30.0 * i, 0.0] for i in range(12)]))):
        with pytest.raises(ssl.ValidationError, match="asynchronous pushes are pending"):
            call()
    # a second async push may queue behind the first
    tk2 = eng.push_samples_async(pcm[:, 2000:])
    with pytest.raises(ssl.ValidationError, match="too small"):
        eng.wait_results(tk2, cap=1)  # refused before anything is consumed
    out = eng.wait_results(tk2)
    assert out["n"] > 1
    eng.push(frames)  # collected: synchronous calls work again
    eng.close()


def test_run_locate_sinks_blocks_before_the_bad_frame(golden):
    from paper_2504_03373_b200 import ssl

    g = golden("c1_band")
    t, ns = int(g["t"]), int(g["ns"])
    x = g["x"].copy()
    k = t + 1
    x[k, 0, 0] = np.nan
    steer = ssl.SteeringField(x.shape[1], 0, x.shape[2] - 1, g["dirs"], g["h"])
    noise = ssl.NoiseModel(ssl.CorrelationSet(x.shape[1], g["k"]))
    seen = []
    with pytest.raises(ssl.ValidationError, match="non-finite"):
        ssl.run_locate(x, t, noise, steer, music=ssl.MusicConfig(num_sources=ns), sink=seen.append)
    assert [f.frame_index for f in seen] == list(range(t - 1, k))
    for b, fe in enumerate(seen):
        c = int(g["count"][b])
        assert [e.direction_index for e in fe.estimates] == list(g["idx"][b][:c])


def test_peak_search_context_never_serves_a_spectrum():
    """calc_average_power after peak_search at m = num_sources + 1, one bin:
    the peak-search context holds placeholder steering vectors, so the
    spectrum must come from its own context (same result before and after)."""
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(5)
    m, ns, d = 3, 2, 12
    x = (rng.standard_normal((6, m)) + 1j * rng.standard_normal((6, m))).astype(np.complex64)
    r = ssl.CorrelationSet(m, (x.T @ x.conj() / 6).astype(np.complex64)[None])
    noise = ssl.NoiseModel.identity(m, 1)
    basis = ssl.gsvd(noise, r)
    dirs = np.array([[30.0 * i, 0.0] for i in range(d)])
    h = (rng.standard_normal((d, 1, m)) + 1j * rng.standard_normal((d, 1, m))).astype(np.complex64)
    steer = ssl.SteeringField(m, 0, 0, dirs, h)
    cfg = ssl.MusicConfig(num_sources=ns)
    p1 = ssl.calc_average_power(basis, steer, cfg).power.copy()
    topo = ssl.DirectionTopology.build(dirs)
    peaks = ssl.peak_search(p1, dirs, topo, cfg)
    assert 0 < len(peaks) <= ns
    p2 = ssl.calc_average_power(basis, steer, cfg).power
    assert np.array_equal(p1, p2)
    assert np.all(p1 > 0)
