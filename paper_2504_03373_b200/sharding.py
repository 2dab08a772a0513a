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

    def push(self, frames: np.ndarray):
        import torch

        results = []
        for c0 in range(0, frames.shape[0], self.max_batch):
            local = np.ascontiguousarray(frames[c0:c0 + self.max_batch, :, self.lo:self.hi])
            with torch.cuda.stream(self.stream):
                n = self.eng.push(local)["n"]  # local-bin estimates are superseded below
                if n == 0:
                    continue
                p_local = torch.empty((n, self.hi - self.lo, self.dirs), dtype=torch.float64, device=self.device)
                self.eng.copy_bin_power_device(p_local.data_ptr(), n)
                self.stream.synchronize()
                p_all = gather_bin_power(p_local, self.slices, self.group)
                self.eng.integrate_peaks_device(p_all.data_ptr(), n, self.bins)
                results.append(self.eng.read_results(n, power=True))
        if not results:
            return dict(n=0)
        out = {k: np.concatenate([r[k] for r in results]) for k in ("frame_index", "count", "idx", "power_est", "low",
                                                                     "power")}
        out["n"] = int(out["count"].shape[0])
        return out
