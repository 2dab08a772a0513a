"""Multi-GPU host logic on CPU (gloo, world size 2).

Bin sharding of one array: each rank computes the per-bin MUSIC powers of its
bin slice (here with the CPU oracle standing in for the device kernels), the
slices are all-gathered and assembled in global bin order, and the ordered
broadband sum + peak search must reproduce the single-process result bit for
bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2504_03373_b200 import sharding

        g = dict(np.load(os.path.join(ROOT, "tests", "golden", name + ".npz")))
        ns = int(g["ns"])
        bins = g["e0"].shape[0]
        slices = sharding.bin_slices(bins, world)
        lo, hi = slices[rank]
        port_ = oracle.port()
        # stand-in for the rank's device spectrum over its bin slice
        _, bp = port_.spectrum(g["e0"][lo:hi], g["h"][:, lo:hi], ns, keep_bins=True, threads=1)
        p_local = torch.from_numpy(bp)[None]  # [n=1][b_local][D]
        p_all = sharding.gather_bin_power(p_local, slices)
        # ordered integration (music.cpp:143-160) as the device kernel does it
        pa = p_all[0].numpy()
        pbar = np.zeros(pa.shape[1])
        for b in range(pa.shape[0]):
            pbar = pbar + pa[b]
        q.put((rank, pa, pbar))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1_band", "c2_band"])
def test_bin_sharded_gather_is_bit_exact(name, port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", name + ".npz")))
    ns = int(g["ns"])
    full_p, full_bp = port.spectrum(g["e0"], g["h"], ns, keep_bins=True, threads=1)
    for rank, pa, pbar in out:
        assert np.array_equal(pa.view(np.uint64), full_bp.view(np.uint64))
        assert np.array_equal(pbar.view(np.uint64), full_p.view(np.uint64))
        # and the same estimates as the reference fixture's first block
        off, nbr = port.topology(g["dirs"], 10.0)
        idx, _, _ = port.peaks(pbar, off, nbr, ns)
        assert np.array_equal(idx, g["idx"][0][: int(g["count"][0])])


def test_bin_slices_cover_and_balance():
    from paper_2504_03373_b200 import sharding

    for bins in (1, 7, 12, 257):
        for world in (1, 2, 3, 8):
            s = sharding.bin_slices(bins, world)
            assert s[0][0] == 0 and s[-1][1] == bins
            assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
            sizes = [hi - lo for lo, hi in s]
            assert max(sizes) - min(sizes) <= 1


def test_pad_and_assemble_roundtrip():
    from paper_2504_03373_b200 import sharding

    rng = np.random.default_rng(0)
    bins, d, n, world = 11, 5, 3, 4
    full = torch.from_numpy(rng.standard_normal((n, bins, d)))
    slices = sharding.bin_slices(bins, world)
    bmax = max(hi - lo for lo, hi in slices)
    gathered = torch.stack([sharding.pad_slice(full[:, lo:hi], bmax) for lo, hi in slices])
    assert torch.equal(sharding.assemble(gathered, slices), full)


@pytest.mark.gpu
def test_bin_sharded_locator_on_one_gpu_matches_engine(golden):
    """The device side of bin sharding (copy-out, NCCL all-gather, ordered
    integration kernel) at world size 1 reproduces the plain engine."""
    from paper_2504_03373_b200 import sharding, ssl

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = golden("c1_band")
        t, ns = int(g["t"]), int(g["ns"])
        m, bins = g["x"].shape[1], g["x"].shape[2]
        loc = sharding.BinShardedLocator(m, bins, g["k"], g["h"], g["dirs"], window_frames=t,
                                         music=ssl.MusicConfig(num_sources=ns), max_batch=8)
        out = loc.push(g["x"])
        assert out["n"] == g["power"].shape[0]
        for b in range(out["n"]):
            assert np.max(np.abs(out["power"][b] - g["power"][b]) / g["power"][b]) <= 1e-9
            c = int(g["count"][b])
            assert np.array_equal(out["idx"][b][:c], g["idx"][b][:c])
    finally:
        dist.destroy_process_group()
