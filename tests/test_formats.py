"""On-disk formats and JSONL records through the C ABI,
against the reference's own readers/writers (oracle/_ref).  Host-only code:
runs without a GPU.

  SSLC tensor files      byte-identical files both ways, identical payloads
  steering files         byte-identical files (header as nlohmann dumps it)
  errors                 the reference's IoError messages
  JSONL records          field-identical to nlohmann::json::dump of the
                         reference's record (pipeline.cpp:268-283): same keys
                         and order, bit-identical values
"""
import json

import numpy as np
import pytest


def rand_k(rng, bins, m):
    return (rng.standard_normal((bins, m, m)) + 1j * rng.standard_normal((bins, m, m))).astype(np.complex64)


def test_correlation_files_round_trip_with_the_reference(ref, tmp_path):
    from paper_2504_03373_b200 import formats

    rng = np.random.default_rng(1)
    k = rand_k(rng, 7, 5)
    ours, theirs = str(tmp_path / "ours.sslc"), str(tmp_path / "ref.sslc")
    formats.save_correlation(ours, k, 42)
    ref.save_correlation(theirs, k, 42)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    got, t = formats.load_correlation(theirs)
    assert t == 42 and got.m == 5 and np.array_equal(got.bins.view(np.uint32), k.view(np.uint32))
    back, t2 = ref.load_correlation(ours)
    assert t2 == 42 and np.array_equal(back.view(np.uint32), k.view(np.uint32))


def test_correlation_file_errors(tmp_path):
    from paper_2504_03373_b200 import formats
    from paper_2504_03373_b200.errors import IoError

    p = str(tmp_path / "x.sslc")
    with pytest.raises(IoError, match="cannot open"):
        formats.load_correlation(str(tmp_path / "missing.sslc"))
    open(p, "wb").write(b"NOPE" + bytes(12))
    with pytest.raises(IoError, match="not a correlation tensor file"):
        formats.load_correlation(p)
    open(p, "wb").write(b"SSLC" + (0).to_bytes(4, "little") + (1).to_bytes(4, "little") + bytes(4))
    with pytest.raises(IoError, match="implausible header"):
        formats.load_correlation(p)
    k = rand_k(np.random.default_rng(2), 3, 4)
    formats.save_correlation(p, k, 5)
    data = open(p, "rb").read()
    open(p, "wb").write(data[:-8])
    with pytest.raises(IoError, match="truncated payload"):
        formats.load_correlation(p)


def test_steering_files_round_trip_with_the_reference(ref, tmp_path):
    from paper_2504_03373_b200 import formats, ssl, synth

    mics = synth.circular(8, 0.05)
    dirs = np.concatenate([synth.azimuth_grid(5.0), [[12.5, -30.0], [0.1, 1e-7], [359.9999999, 45.25]]])
    h = synth.steering(mics, dirs, 16, 20)
    ours, theirs = str(tmp_path / "ours.steer"), str(tmp_path / "ref.steer")
    formats.save_steering(ours, ssl.SteeringField(8, 16, 20, dirs, h))
    ref.save_steering(theirs, 8, 16, 20, dirs, h)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    f = formats.load_steering(theirs)
    assert (f.m, f.bin_min, f.bin_max) == (8, 16, 20)
    assert np.array_equal(f.directions, dirs) and np.array_equal(f.vectors.view(np.uint32), h.view(np.uint32))
    m, lo, hi, d2, h2 = ref.load_steering(ours)
    assert (m, lo, hi) == (8, 16, 20) and np.array_equal(d2, dirs) and np.array_equal(h2, h)


def test_steering_file_errors(tmp_path):
    from paper_2504_03373_b200 import formats
    from paper_2504_03373_b200.errors import IoError

    p = str(tmp_path / "s.steer")
    open(p, "wb").write(b"")
    with pytest.raises(IoError, match="missing header line"):
        formats.load_steering(p)
    open(p, "wb").write(b'{"m": 2, "bin_min": 0}\n')
    with pytest.raises(IoError, match="bad steering header"):
        formats.load_steering(p)
    open(p, "wb").write(b'{"m": 2, "bin_min": 3, "bin_max": 1, "directions": [[0, 0]]}\n')
    with pytest.raises(IoError, match="bad steering header"):
        formats.load_steering(p)
    open(p, "wb").write(b'{"m": 2, "bin_min": 0, "bin_max": 0, "directions": [[0, 0]]}\n' + bytes(8))
    with pytest.raises(IoError, match="truncated steering payload"):
        formats.load_steering(p)


def _records(rng, n):
    dirs = np.concatenate([np.stack([np.arange(72) * 5.0, np.zeros(72)], 1),
                           [[12.5, -30.0], [0.1, 1e-7], [359.99999999999994, 45.25], [1e20, -1e-5]]])
    vals = [0.0, 1.0, 40.0, 1e-5, 1.5e-5, 9.999e-5, 0.0001, 123456789012345.0, 1234567890123456.0, 1e15, 1e16,
            2.5e-300, 1.7976931348623157e308, 5e-324, 1 / 3, 2 / 3, 0.1, 0.3, 1e-4, 0.001234]
    for _ in range(n):
        c = int(rng.integers(0, 4))
        idx = rng.integers(0, len(dirs), c).astype(np.uint32)
        pw = np.array([vals[int(rng.integers(0, len(vals)))] * (1 if rng.random() < 0.8 else -1) if rng.random() < 0.5
                       else float(np.exp(rng.uniform(-60, 60))) for _ in range(c)])
        low = (rng.random(c) < 0.3).astype(np.uint8)
        yield int(rng.integers(0, 2**40)), idx, dirs, pw, low


def test_jsonl_records_match_nlohmann(ref):
    """Field-level parity: the same keys in the same order, the same values
    to the bit (every number is a round-trip-exact spelling).  The text is
    identical too except where nlohmann's Grisu2 picks a longer (17-digit)
    spelling of the same double than the shortest one written here."""
    from paper_2504_03373_b200 import formats, ssl

    rng = np.random.default_rng(7)
    same_text = 0
    n = 2000
    for frame, idx, dirs, pw, low in _records(rng, n):
        ests = [ssl.SourceEstimate(int(j), ssl.Direction(*dirs[j]), float(p), bool(lo)) for j, p, lo in
                zip(idx, pw, low)]
        ours = formats.format_estimates_json(frame, ests, dirs)
        theirs = ref.format_estimates(frame, idx, dirs, pw, low)
        a, b = json.loads(ours), json.loads(theirs)
        assert a == b, (ours, theirs)
        assert list(a) == list(b) == ["estimates", "frame"]
        for ea, eb in zip(a["estimates"], b["estimates"]):
            assert list(ea) == list(eb)
        same_text += ours == theirs
    assert same_text >= 0.95 * n
