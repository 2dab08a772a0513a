"""The C-ABI boundary without a GPU: the library loads, exports every entry
point include/sslgpu.h declares, refuses to run without a device (no CPU
fallback), and its host-side helpers (topology) match the reference."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sslgpu.h")).read()
    return sorted(set(re.findall(r"\b(sslg_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_2504_03373_b200 import _capi

    assert set(header_symbols()) == set(_capi.EXPORTS)


def test_library_exports_every_header_symbol():
    from paper_2504_03373_b200 import _capi

    L = _capi.load()
    for name in header_symbols():
        assert hasattr(L, name), name


def test_no_cpu_fallback_without_device():
    from conftest import gpu_available

    if gpu_available():
        pytest.skip("a device is present")
    from paper_2504_03373_b200 import ssl

    with pytest.raises(ssl.DeviceError, match="no CPU fallback"):
        ssl.Engine(8, 4)


def test_config_defaults_follow_reference():
    from paper_2504_03373_b200 import _capi

    cfg = _capi.Config()
    _capi.load().sslg_config_default(C.byref(cfg))
    # pipeline.hpp:23 (T = 50), music.hpp:49-62, gsvd.hpp:14-26, correlation.hpp:31
    assert cfg.window_frames == 50 and cfg.rebuild_interval == 1000
    assert cfg.num_sources == 1 and cfg.low_power_ratio == pytest.approx(1.25)
    assert cfg.denominator_floor == pytest.approx(1e-12) and cfg.squared_denominator == 0
    assert cfg.pivoting == 1 and cfg.canonical_subspaces == 1


@pytest.mark.parametrize("radius", [10.0, 11.0, 6.0])
def test_host_topology_matches_reference(port, radius):
    """DirectionTopology::build (music.cpp:176-195); the 72-azimuth ring at
    exactly 10 degrees is rounding-dependent and asymmetric."""
    from paper_2504_03373_b200 import ssl

    dirs = np.array([[i * 5.0, 0.0] for i in range(72)])
    t = ssl.DirectionTopology.build(dirs, radius)
    off, nbr = port.topology(dirs, radius)
    assert np.array_equal(t.offsets, off) and np.array_equal(t.nbr, nbr)
    if radius == 10.0:
        assert sorted(t.neighbors[0]) == [1, 2, 71]
        assert sorted(t.neighbors[36]) == [34, 35, 37, 38]


def test_host_topology_sphere_and_azel(port):
    from paper_2504_03373_b200 import ssl, synth

    for dirs in (synth.azel_grid(5.0), ):
        t = ssl.DirectionTopology.build(dirs, 10.0)
        off, nbr = port.topology(dirs, 10.0)
        assert np.array_equal(t.offsets, off) and np.array_equal(t.nbr, nbr)


def test_topology_capacity_error():
    from paper_2504_03373_b200 import _capi

    L = _capi.load()
    dirs = np.array([[0.0, 0.0], [1.0, 0.0]])
    off = np.zeros(3, np.uint32)
    need = C.c_uint32()
    rc = L.sslg_build_topology(_capi.f64p(dirs), 2, 10.0, _capi.u32p(off), None, 0, C.byref(need))
    assert rc == _capi.SSLG_VALIDATION and need.value == 2


def test_sources_are_sm100a_only():
    from paper_2504_03373_b200 import build

    assert "arch=compute_100a,code=sm_100a" in " ".join(build.NVCC_FLAGS)
    for f in os.listdir(build.CSRC):
        if f.endswith(".cu"):
            txt = open(os.path.join(build.CSRC, f)).read()
            assert "oracle" not in txt.lower() or "oracle algorithm" in txt.lower(), f
