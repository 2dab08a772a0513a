"""Multi-GPU scheduling of the hot path.

Two partitions, one process per GPU (torch.distributed for the plumbing):

* **streams/arrays** — every rank runs whole arrays; no data-path collective
  (`bench.py --gpus N`, weak scaling).
* **bins of one array** — rank r owns a contiguous slice of frequency bins:
  its correlation window, GSVD and per-bin MUSIC powers cover only those bins.
  One all-gather of the per-bin powers P[n][b_r][D] (padded to equal slices,
  ~9.5 KB per rank per block at G = 8, D = 72) rebuilds P[n][B][D] in global
  bin order on every rank, and the device integration kernel sums it in
  ascending bin order (music.cpp:143-160) — bit-identical to one GPU.  An
  all-reduce of partial FP64 sums is deliberately avoided: its association
  order would differ from the sequential sum and could break exact ties
  between directions (music.cpp:215-223).

The slice/pad/assemble functions are plain tensor code so the gather order is
testable with the gloo backend on CPU (tests/test_sharding.py).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def bin_slices(bins: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous [lo, hi) slices, sizes differing by at most one."""
    base, extra = divmod(bins, world)
    out, lo = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((lo, lo + n))
        lo += n
    return out


def pad_slice(p_local, bmax: int):
    """[n][b][D] -> [n][bmax][D] (zero rows after the slice)."""
    import torch

    n, b, d = p_local.shape
    if b == bmax:
        return p_local.contiguous()
    out = torch.zeros((n, bmax, d), dtype=p_local.dtype, device=p_local.device)
    out[:, :b] = p_local
    return out


def assemble(gathered, slices: Sequence[Tuple[int, int]]):
    """[world][n][bmax][D] gathered slices -> [n][B][D] in global bin order."""
    import torch

    parts = [gathered[r, :, : hi - lo] for r, (lo, hi) in enumerate(slices)]
    return torch.cat(parts, dim=1).contiguous()


def gather_bin_power(p_local, slices: Sequence[Tuple[int, int]], group=None):
    """All-gather every rank's per-bin powers and assemble them in bin order."""
    import torch
    import torch.distributed as dist

    world = len(slices)
    bmax = max(hi - lo for lo, hi in slices)
    padded = pad_slice(p_local, bmax)
    out = torch.empty((world,) + tuple(padded.shape), dtype=padded.dtype, device=padded.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, padded, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), padded, group=group)
    return assemble(out, slices)


class BinShardedLocator:
    """One array's bins spread over the ranks of `group` (one GPU per rank).

    push(frames [F][m][B] complex64, host) -> dict of the n emitted blocks'
    estimates and broadband power, identical on every rank.
    """

    def __init__(self, m: int, bins: int, k: np.ndarray, h: np.ndarray, dirs: np.ndarray, window_frames: int = 50,
                 music=None, solver=None, max_batch: int = 16, device: int = 0, group=None):
        import torch
        import torch.distributed as dist

        from . import ssl

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        self.slices = bin_slices(bins, self.world)
        self.lo, self.hi = self.slices[self.rank]
        self.bins, self.dirs = bins, h.shape[0]
        self.device = device
        self.stream = torch.cuda.Stream(device)
        topo = ssl.DirectionTopology.build(dirs)
        self.eng = ssl.Engine(m, self.hi - self.lo, window_frames=window_frames, music=music, solver=solver,
                              max_batch=max_batch, device=device, stream=self.stream.cuda_stream)
        self.eng.set_noise_model(np.ascontiguousarray(k[self.lo:self.hi]))
        self.eng.set_steering(np.ascontiguousarray(h[:, self.lo:self.hi]), dirs, topo)
        self.max_batch = max_batch
        self.pushed = 0

    def push(self, frames: np.ndarray):
        """frames [F][m][B] complex64 (host).  The rank's bin slice goes to the
        device in one copy; the pushes, the per-bin power copies, ONE
        all-gather for every block of the call and the ordered integration
        are all stream-ordered on the locator's stream -- the host waits only
        when the estimates are read back."""
        import torch

        frames = np.ascontiguousarray(frames, np.complex64)
        nfr = frames.shape[0]
        pushed0 = self.pushed
        self.pushed += nfr
        if nfr == 0:
            return dict(n=0)
        local = np.ascontiguousarray(frames[:, :, self.lo:self.hi])
        b_local = self.hi - self.lo
        with torch.cuda.stream(self.stream):
            x = torch.from_numpy(local.view(np.float32)).pin_memory().to(f"cuda:{self.device}", non_blocking=True)
            chunks = []
            for c0 in range(0, nfr, self.max_batch):
                nf = min(self.max_batch, nfr - c0)
                n = self.eng.push_device(x[c0:c0 + nf].data_ptr(), nf)  # no host synchronization
                if n:
                    p = torch.empty((n, b_local, self.dirs), dtype=torch.float64, device=self.device)
                    self.eng.copy_bin_power_device(p.data_ptr(), n)
                    chunks.append(p)
            if not chunks:
                return dict(n=0)
            p_local = chunks[0] if len(chunks) == 1 else torch.cat(chunks)
            p_all = gather_bin_power(p_local, self.slices, self.group)  # one collective per push
            results = []
            for c0 in range(0, p_all.shape[0], self.max_batch):
                n = min(self.max_batch, p_all.shape[0] - c0)
                self.eng.integrate_peaks_device(p_all[c0:c0 + n].data_ptr(), n, self.bins)
                results.append(self.eng.read_results(n, power=True))
        out = {k: np.concatenate([r[k] for r in results]) for k in ("count", "idx", "power_est", "low", "power")}
        n = int(out["count"].shape[0])
        out["n"] = n
        out["frame_index"] = np.arange(pushed0 + nfr - n, pushed0 + nfr, dtype=np.uint32)
        return out
