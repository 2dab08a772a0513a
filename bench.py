#!/usr/bin/env python
"""Throughput of the B200 GSVD-MUSIC hot path (BASELINE.json metric):
60-ch GSVD-MUSIC SSL blocks/sec, GSVD latency per block (us), x real-time.

Workload (BASELINE.json configs[2], "C3"): 60-ch circular array (r = 0.3 m),
16 kHz, 512-pt FFT -> 257 bins, 72 azimuths, two targets under four rotor
noise sources + diffuse floor, K captured from noise-only frames, T = 50,
Ns = 2.  Synthetic STFT-domain frames (paper_2504_03373_b200/synth.py).

One step = one pass of the hot path over one batch of `--batch` new STFT
frames per GPU = `--batch` blocks (the window is kept full), each block being
correlation update + GSVD over 257 bins + MUSIC over 72 x 257 + integration +
peak search.  N > 1: one independent array (stream) per GPU, no data-path
collective ("scaling": "weak"); time = max over ranks of the device time.

Arms:
  default            this engine (libsslgpu.so); prints one JSON line
  --impl reference   the reference's own CPU implementation (oracle/_ref, the
                     unmodified sslkit library) on the host cores, same
                     workload / metric; rank 0 only
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "60-ch GSVD-MUSIC SSL blocks/sec; GSVD latency per block (us); x real-time"
UNIT = "blocks/s"
REALTIME_BLOCKS_PER_S = 100.0  # fs / shift = 16000 / 160 per array


WORKLOADS = {"c1": "C1 (BASELINE configs[0])", "c2": "C2 (BASELINE configs[1])", "c3": "C3 (BASELINE configs[2])",
             "c4": "C4 (BASELINE configs[3], 72 az x 19 el grid)"}


def scene_label(args, w):
    from paper_2504_03373_b200 import synth

    return f"{WORKLOADS[args.config]}: {synth.describe(args.config)}"


def frames_from_pcm(w):
    """The scene's STFT frames for the CPU arms (oracle restatement of
    stft_stream, bit-identical to the reference and to the device STFT)."""
    import oracle

    return oracle.port().stft(w.pcm, w.frame_length, w.shift, 0, w.bin_min, w.bin_max)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=32, help="blocks (new frames) per step per GPU")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-blocks", type=int, default=48)
    p.add_argument("--no-flush", action="store_true")
    p.add_argument("--shard", default="arrays", choices=["arrays", "bins"],
                   help="N>1: one array per GPU (weak) or one array's bins split over the GPUs with an all-gather "
                        "of per-bin powers (strong, BinShardedLocator)")
    p.add_argument("--arrays", type=int, default=1,
                   help="independent arrays (engines, one stream each) per GPU; >1 = BASELINE configs[4] (C5)")
    p.add_argument("--dry-run", action="store_true",
                   help="launcher/plumbing check without a GPU: gloo ranks, barrier + max-over-ranks timing of an "
                        "empty step, the JSON line with n_gpus (tests/test_bench_contract.py)")
    return p.parse_args()


def relaunch_if_needed(args) -> bool:
    """`python bench.py --gpus N` (N > 1) outside torchrun starts the N
    ranks itself: it re-executes under torch.distributed.run with one process
    per GPU (127.0.0.1 rendezvous), forwards every argument and exits with the
    launcher's status.  Under torchrun (WORLD_SIZE set) nothing happens."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


def run_dry(args, rank, world):
    """The multi-rank plumbing of the bench without a device: gloo process
    group, barrier, an (empty) timed step per step, max over ranks, one JSON
    line from rank 0 naming every rank that took part."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
    ms = (time.perf_counter() - t0) * 1e3
    ranks = [rank]
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        got = [None] * world
        dist.all_gather_object(got, rank)
        ranks = got
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / max(1, args.steps), "dry_run": True,
                          "ranks": ranks, "scaling": "weak"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------


class ClockSampler:
    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self._ok = False

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self._ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# algorithmic work per block (SURVEY.md §8(d) convention)
# ---------------------------------------------------------------------------


def algorithmic(m, bins, dirs, ns, t=50):
    s_nom = 10
    f_whiten = 8.0 * bins * m ** 3
    f_jacobi = bins * s_nom * m * (m - 1) / 2 * 36 * m
    f_music = 8.0 * dirs * bins * (m - ns) * m
    corr_bytes = 2 * bins * m * 8 + bins * m * m * 8
    spec_bytes = bins * (m - ns) * m * 16 + bins * dirs * m * 8 + bins * dirs * 8
    return dict(f_whiten=f_whiten, f_jacobi=f_jacobi, f_music=f_music, corr_bytes=corr_bytes, spec_bytes=spec_bytes)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(path):
        try:
            with open(path) as f:
                return json.load(f)
        except Exception:
            return None
    return None


# ---------------------------------------------------------------------------
# reference CPU arm / cpu_baseline leg (oracle/_ref = the unmodified reference)
# ---------------------------------------------------------------------------


def reference_time_blocks(w, nblocks, threads):
    """Times the reference's run_locate per-frame loop (pipeline.cpp:227-245,
    batched float path, `threads` workers) over `nblocks` emitted blocks of the
    workload; returns (seconds per block, stage seconds)."""
    import oracle

    R = oracle.ref()
    frames = w.t - 1 + nblocks
    wl = oracle.Workload(w.x[:frames], w.k, w.h, w.dirs)
    mc = oracle.MusicCfg.make(num_sources=w.ns)
    out = R.locate_frames(wl, w.t, mc, path=0, threads=threads)
    st = out["stage_s"]
    # stage clocks of the emitting frames: push + normalize + gsvd + spectrum
    # + peaks per block (the T-1 window-filling pushes are not charged)
    return float(np.sum(st)) / nblocks, st, out


def run_reference_arm(args, w, rank, world):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    per_step = max(1, min(args.batch, 4))
    for _ in range(max(0, args.warmup)):
        reference_time_blocks(w, per_step, cores)
    times = []
    for _ in range(args.steps):
        spb, _, _ = reference_time_blocks(w, per_step, cores)
        times.append(spb * per_step)
    total = sum(times)
    value = args.steps * per_step / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": scene_label(args, w),
                   "blocks_per_step": per_step, "path": "ssl::gsvd batched float + calc_average_power<float>",
                   "input": "STFT frames of the same PCM (the reference's own STFT is not timed)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{per_step} blocks per step of the same C3 stream through the reference "
                                   f"run_locate loop (oracle/_ref, {cores} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "x_realtime": value / REALTIME_BLOCKS_PER_S,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------


def main():
    args = parse()
    relaunch_if_needed(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        run_dry(args, rank, world)
        return

    from paper_2504_03373_b200 import synth

    # the scene as PCM (SampleBlock): the product path runs the device STFT
    # front end; the reference arm and the cpu_baseline see the same frames
    frames_needed = 50 + (args.warmup + args.steps + 1) * args.batch + 8
    w = synth.make_pcm(args.config, duration_s=((frames_needed - 1) * 160 + 512) / 16000.0, seed=11 + rank)

    if args.impl == "reference":
        try:
            import oracle

            if not oracle.ref_available():
                raise FileNotFoundError("oracle/_ref/libsslref.so missing")
        except Exception as e:  # the reference arm is unavailable
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": str(e).splitlines()[0]}), flush=True)
            return
        w.x = frames_from_pcm(w)
        run_reference_arm(args, w, rank, world)
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    device = local

    from paper_2504_03373_b200 import _capi, ssl

    if args.arrays > 1:
        run_arrays(args, w, rank, world, device, dist)
        return
    if args.shard == "bins":
        run_bin_sharded(args, w, rank, world, device, dist)
        return

    # a dedicated stream: the engine launches on it and the CUDA events below
    # are recorded on it (torch's default stream is the legacy NULL stream)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    eng = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns),
                     max_batch=args.batch, device=device, stream=stream.cuda_stream)
    eng.set_noise_model(w.k)
    eng.set_steering(w.h, w.dirs)
    eng.set_stft(ssl.StftConfig(w.frame_length, w.shift, "hann", w.bin_min, w.bin_max))
    w.x = eng.stft(w.pcm)  # the device STFT of the scene (bit-identical to the reference's)

    # inputs resident in HBM before the timed region
    x_all = torch.from_numpy(w.x.view(np.float32)).to(f"cuda:{device}")  # [F][m][bins*2]
    fsz = w.m * w.bins
    pos = 0

    def next_frames(n):
        nonlocal pos
        if pos + n > x_all.shape[0]:
            pos = w.t  # recycle the pool after the fill
        v = x_all[pos:pos + n]
        pos += n
        return v

    # fill the window (frames 0..T-2), then one emitting push
    left = w.t - 1
    while left > 0:
        nf = min(left, args.batch)
        fill = next_frames(nf)
        eng.push_device(fill.data_ptr(), nf)
        left -= nf
    flush_buf = None if args.no_flush else torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)

    def sync_all():
        torch.cuda.synchronize(device)
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        xb = next_frames(args.batch)
        eng.push_device(xb.data_ptr(), args.batch)
    sync_all()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stage = np.zeros(5)
    launches = 0
    emitted = 0
    with ClockSampler(device) as clk:
        for i in range(args.steps):
            xb = next_frames(args.batch)
            if flush_buf is not None:
                flush_buf.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            n = eng.push_device(xb.data_ptr(), args.batch)
            ev[i][1].record(stream)
            stream.synchronize()
            stage += eng.stage_ms()
            launches += eng.launch_count()
            emitted += n
        sync_all()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    if dist is not None:
        t = torch.tensor([total_ms], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        e = torch.tensor([emitted], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        emitted_all = int(e.item())
    else:
        emitted_all = emitted
    value = emitted_all / (total_ms * 1e-3)
    res = eng.read_results(args.batch, sigma=False)
    hits = float(np.mean([set(r[: c].tolist()) == set(w.targets) for r, c in zip(res["idx"], res["count"])]))
    # fraction of the targets among each block's peaks (on the C4 3D grid
    # the reference's own peak search ranks an elevation sidelobe of one
    # target, 10 deg off -- outside the neighbour test -- above another target)
    recall = float(np.mean([len(set(r[: c].tolist()) & set(w.targets)) / len(w.targets)
                            for r, c in zip(res["idx"], res["count"])]))

    # single-block GSVD latency (one array, one block per launch)
    lat = []
    for _ in range(5):
        xb = next_frames(1)
        eng.push_device(xb.data_ptr(), 1)
        eng.synchronize()
        s = eng.stage_ms()
        lat.append(1e3 * float(s[1] + s[2]))
    gsvd_latency_us = float(np.median(lat))

    # e2e: run_locate's public entry on SampleBlocks (sslg_push_samples): per
    # step, batch * shift new samples per channel from pinned host memory go
    # H2D, the device STFT turns them into frames inside the window, the hot
    # path runs, and the estimates come back D2H -- all inside the timed region
    eng.reset_window()
    step_samples = args.batch * w.shift
    lead = (w.t - 1) * w.shift + w.frame_length - w.shift  # fills the window to T-1 frames
    nchunks = args.warmup + args.steps
    need = lead + nchunks * step_samples
    src = w.pcm if w.pcm.shape[1] >= need else np.tile(w.pcm, (1, need // w.pcm.shape[1] + 1))
    chunks = [torch.from_numpy(np.ascontiguousarray(src[:, lead + i * step_samples:lead + (i + 1) * step_samples]))
              .pin_memory() for i in range(nchunks)]
    eng.push_samples(np.ascontiguousarray(src[:, :lead]))
    e2e_ms = []
    ns = w.ns
    for i in range(nchunks):  # synchronous: one push, wait for its estimates
        xh = chunks[i].numpy()
        sync_all()
        t0 = time.perf_counter()
        out = eng.push_samples(xh)
        dt = time.perf_counter() - t0
        assert out["n"] == args.batch
        if i >= args.warmup:
            e2e_ms.append(dt * 1e3)
    e2e_sync_total = float(sum(e2e_ms))
    # pipelined (sslg_push_samples_async): the next push's H2D, STFT and hot
    # path are queued while the host collects the previous push's estimates
    eng.reset_window()
    eng.push_samples(np.ascontiguousarray(src[:, :lead]))
    for i in range(args.warmup):
        eng.wait_results(eng.push_samples_async(chunks[i].numpy()))
    sync_all()
    t0 = time.perf_counter()
    prev = None
    got = 0
    for i in range(args.warmup, nchunks):
        t = eng.push_samples_async(chunks[i].numpy())
        if prev is not None:
            got += eng.wait_results(prev)["n"]
        prev = t
    got += eng.wait_results(prev)["n"]
    e2e_total = (time.perf_counter() - t0) * 1e3
    assert got == args.steps * args.batch
    if dist is not None:
        t = torch.tensor([e2e_total, e2e_sync_total], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total, e2e_sync_total = float(t[0].item()), float(t[1].item())
    e2e_value = world * args.steps * args.batch / (e2e_total * 1e-3)
    e2e_sync_value = world * args.steps * args.batch / (e2e_sync_total * 1e-3)
    h2d = w.m * step_samples * 4
    d2h = args.batch * (ns * (4 + 8 + 1) + 4)  # idx u32, power f64, low u8 per estimate; count u32 per block

    if rank == 0:
        alg = algorithmic(w.m, w.bins, w.h.shape[0], w.ns, w.t)
        blocks_per_launch = args.batch
        jac_ms = stage[1] / args.steps
        can_ms = stage[2] / args.steps
        spec_ms = stage[3] / args.steps
        corr_ms = stage[0] / args.steps
        fp64 = ctypes_probe(device)
        fp32 = ctypes_probe(device, fp32=True)
        peaks, peak_kind = load_peaks()
        achieved_tf = (alg["f_whiten"] + alg["f_jacobi"]) * blocks_per_launch / (jac_ms * 1e-3) / 1e12
        traffic = load_traffic()
        jac_traffic = None
        # this config's own ncu capture (profiles/ncu_summary.json, keys "<config>:<kernel>"), per block, scaled
        # to this launch; no capture of this config -> null (never another config's numbers)
        parts = (["jacobi_prologue", "sweep_bip_kernel", "jacobi_epilogue"] if w.m == 60
                 else ["small_jacobi_kernel"] if w.m <= 16 else ["jacobi_kernel"])
        keys = [f"{args.config}:{k}" for k in parts]
        if traffic and all(k in traffic for k in keys):
            jac_traffic = sum(traffic[k]["dram_bytes_per_launch"] / traffic[k].get("blocks_per_launch", 8)
                              for k in keys) * blocks_per_launch
        roofline = {
            "kernel": ("GSVD solver: jacobi_kernel<60,1> (whitening A = K^-1 R + QRCP) -> sweep_bip_kernel "
                       "(FP64 one-sided Jacobi sweeps) -> jacobi_kernel<60,3> (sigma, back-multiply, "
                       "canonical bases); achieved over the three launches" if w.m == 60 else
                       "GSVD solver: small_jacobi_kernel (one lane group per bin: whitening, one-sided Jacobi, "
                       "sort, canonical bases)" if w.m <= 16 else "GSVD solver: jacobi_kernel"),
            "bound": "fp64", "achieved": achieved_tf, "peak": fp64, "unit": "TFLOP/s",
            "frac": achieved_tf / fp64 if fp64 else None, "traffic": jac_traffic,
            # the same achieved rate against the FP32 FMA ceiling (what a float
            # Jacobi could at most reach; the solver computes in FP64)
            "fp32_peak": fp32, "frac_vs_fp32_peak": achieved_tf / fp32 if fp32 else None,
            "peak_kind": "measured in-run (DFMA microbenchmark, sslg_probe_fp64_tflops); "
                         "MEASURED_PEAKS.json has no FP64 entry",
            "flops_per_block": alg["f_whiten"] + alg["f_jacobi"],
            "flop_convention": "SURVEY.md §8(d): 8*B*M^3 + B*10*M(M-1)/2*36M",
        }
        kernels = {
            "correlation": {"ms_per_launch": corr_ms,
                            "achieved_gbs": alg["corr_bytes"] * blocks_per_launch / (corr_ms * 1e-3) / 1e9,
                            "peak_gbs": peaks.get("hbm_gbs"), "peak_kind": peak_kind},
            "jacobi": {"ms_per_launch": jac_ms, "us_per_block": 1e3 * jac_ms / blocks_per_launch},
            "canonical": {"ms_per_launch": can_ms, "us_per_block": 1e3 * can_ms / blocks_per_launch},
            "spectrum": {"ms_per_launch": spec_ms,
                         "achieved_gbs": alg["spec_bytes"] * blocks_per_launch / (spec_ms * 1e-3) / 1e9,
                         "achieved_tflops": alg["f_music"] * blocks_per_launch / (spec_ms * 1e-3) / 1e12,
                         "peak_gbs": peaks.get("hbm_gbs")},
            "peaks": {"ms_per_launch": stage[4] / args.steps},
        }
        cpu = None
        parity = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(w, args.cpu_sample_blocks)
            if cpu is not None:
                ref_out = cpu.pop("_ref_out")
                def fresh_engine():
                    e = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns),
                                   max_batch=args.batch, device=device)
                    e.set_noise_model(w.k)
                    e.set_steering(w.h, w.dirs)
                    return e

                parity = parity_in_run(w, fresh_engine, ref_out, args.cpu_sample_blocks)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": scene_label(args, w),
                       "input": "PCM; value: frames from the device STFT resident in HBM; e2e: PCM from pinned host",
                       "blocks_per_step_per_gpu": args.batch, "arrays": world,
                       "l2": "flushed (256 MiB write) between timed steps" if not args.no_flush else "not flushed",
                       "parallelism": f"array-sharded x{world} (no data-path collective)"},
            "gsvd_us_per_block": 1e3 * (jac_ms + can_ms) / blocks_per_launch,
            "gsvd_speedup_vs_reference": None if not cpu else {
                "vs_1thread": cpu["gsvd_1thread_us"] / (1e3 * (jac_ms + can_ms) / blocks_per_launch),
                "vs_allcore": cpu["gsvd_allcore_us"] / (1e3 * (jac_ms + can_ms) / blocks_per_launch),
                "reference": "ssl::gsvd (batched float path) per block, noise inverses prepared outside the timer "
                             "(bench.cpp:198-231), median of 5 calls x 5 blocks after a warm-up"},
            "gsvd_latency_us_single_block": gsvd_latency_us,
            "x_realtime": value / REALTIME_BLOCKS_PER_S,
            "target_hit_rate": hits,
            "target_recall": recall,
            "roofline": roofline,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "sslg_push_samples_async + sslg_wait_results (run_locate streaming on pinned host "
                           "PCM: H2D, device STFT, hot path, estimates D2H; one push in flight while the previous "
                           "one is collected); wall clock",
                    "sync_value": e2e_sync_value},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


def run_arrays(args, w, rank, world, device, dist):
    """C5 (BASELINE configs[4]): `--arrays` independent 60-ch arrays per GPU,
    one engine context and one CUDA stream per array, all pushing `--batch`
    new frames per step concurrently; device time from an event on a fork
    stream to the join of every array's stream, max over ranks."""
    import torch

    from paper_2504_03373_b200 import ssl

    A = args.arrays
    main = torch.cuda.Stream(device)
    streams = [torch.cuda.Stream(device) for _ in range(A)]
    engines = []
    for i in range(A):
        e = ssl.Engine(w.m, w.bins, window_frames=w.t, music=ssl.MusicConfig(num_sources=w.ns), max_batch=args.batch,
                       device=device, stream=streams[i].cuda_stream)
        e.set_noise_model(w.k)
        e.set_steering(w.h, w.dirs)
        engines.append(e)
    engines[0].set_stft(ssl.StftConfig(w.frame_length, w.shift, "hann", w.bin_min, w.bin_max))
    x = engines[0].stft(w.pcm)
    x_all = torch.from_numpy(x.view(np.float32)).to(f"cuda:{device}")
    nfr = x_all.shape[0]
    pos = [(17 * i) % max(1, nfr - w.t - args.batch) for i in range(A)]  # each array at its own point in the scene

    def frames(i, n):
        if pos[i] + n > nfr:
            pos[i] = 0
        v = x_all[pos[i]:pos[i] + n]
        pos[i] += n
        return v

    for i, e in enumerate(engines):  # fill every window
        left = w.t - 1
        while left > 0:
            nf = min(left, args.batch)
            e.push_device(frames(i, nf).data_ptr(), nf)
            left -= nf
    torch.cuda.synchronize(device)
    if dist is not None:
        dist.barrier()

    def step(timed):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(main)
        n = 0
        for i, e in enumerate(engines):
            streams[i].wait_event(ev0)
            n += e.push_device(frames(i, args.batch).data_ptr(), args.batch)
        for i in range(A):
            done = torch.cuda.Event()
            done.record(streams[i])
            main.wait_event(done)
        ev1.record(main)
        return ev0, ev1, n

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize(device)
    evs, emitted = [], 0
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            a, b, n = step(True)
            evs.append((a, b))
            emitted += n
        torch.cuda.synchronize(device)
    total_ms = float(sum(a.elapsed_time(b) for a, b in evs))
    if dist is not None:
        t = torch.tensor([total_ms], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        e = torch.tensor([emitted], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        emitted = int(e.item())
    value = emitted / (total_ms * 1e-3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5 (BASELINE configs[4]): {A} concurrent {w.m}-ch arrays per GPU "
                                   f"({WORKLOADS[args.config]} scene), one engine + stream per array",
                       "arrays_per_gpu": A, "blocks_per_step_per_array": args.batch,
                       "parallelism": f"arrays sharded over {world} GPU(s), no data-path collective"},
            "x_realtime_per_array": value / (A * world) / REALTIME_BLOCKS_PER_S,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    for e in engines:
        e.close()
    if dist is not None:
        dist.destroy_process_group()


def run_bin_sharded(args, w, rank, world, device, dist):
    """One array, its 257 bins split over the ranks: per push
    every rank runs correlation + GSVD + per-bin MUSIC on its bin slice, one
    NCCL all-gather of the per-bin powers rebuilds P[n][B][D] in bin order and
    every rank integrates and peak-picks it (bit-identical to one GPU).  Value
    = that array's blocks/s ("scaling": "strong")."""
    import torch

    from paper_2504_03373_b200 import ssl
    from paper_2504_03373_b200.sharding import BinShardedLocator

    if dist is None:  # single process: a one-rank group so the same code path runs
        import torch.distributed as tdist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", device))
        dist = tdist
    e0 = ssl.Engine(w.m, w.bins, max_batch=args.batch, device=device)
    e0.set_stft(ssl.StftConfig(w.frame_length, w.shift, "hann", w.bin_min, w.bin_max))
    x = e0.stft(w.pcm)
    e0.close()
    loc = BinShardedLocator(w.m, w.bins, w.k, w.h, w.dirs, window_frames=w.t,
                            music=ssl.MusicConfig(num_sources=w.ns), max_batch=args.batch, device=device)
    pos = [0]

    def frames(n):
        if pos[0] + n > x.shape[0]:
            pos[0] = w.t
        v = x[pos[0]:pos[0] + n]
        pos[0] += n
        return v

    loc.push(frames(w.t - 1))
    for _ in range(args.warmup):
        loc.push(frames(args.batch))
    torch.cuda.synchronize(device)
    dist.barrier()
    ms, emitted = [], 0
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(loc.stream)
            out = loc.push(frames(args.batch))
            b.record(loc.stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
            emitted += out["n"]
    total = torch.tensor([float(sum(ms))], device=f"cuda:{device}")
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    total_ms = float(total.item())
    value = emitted / (total_ms * 1e-3)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{WORKLOADS[args.config]}: one array, bins sharded over {world} GPU(s)",
                       "bins_per_rank": [hi - lo for lo, hi in loc.slices], "blocks_per_step": args.batch,
                       "parallelism": f"bin-sharded x{world}, one all-gather of per-bin powers per push"},
            "x_realtime": value / REALTIME_BLOCKS_PER_S, "clocks": clk.summary()}), flush=True)
    dist.destroy_process_group()


def ctypes_probe(device, fp32=False):
    import ctypes as C

    from paper_2504_03373_b200 import _capi

    out = C.c_double()
    L = _capi.load()
    rc = (L.sslg_probe_fp32_tflops if fp32 else L.sslg_probe_fp64_tflops)(device, C.byref(out))
    return out.value if rc == 0 else None


def host_cpu_info():
    """CPU model, logical cores and SMT of the host the CPU legs run on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    smt = None
    try:
        with open("/sys/devices/system/cpu/smt/active") as f:
            smt = f.read().strip() == "1"
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": usable, "logical_cpus": os.cpu_count(), "smt_active": smt}


def cpu_baseline(w, nblocks, gsvd_blocks=5, repeats=5):
    """The reference on the host cores (SURVEY §8(d) "CPU baseline beside
    it"): the run_locate loop over `nblocks` blocks with every core, plus the
    stage timings of bench.cpp:198-231 -- ssl::gsvd at 1 thread (the paper's
    "naive" methodology) and at all cores, calc_average_power<float> at 1 and
    all cores -- each with the noise inverses prepared OUTSIDE the timer
    (bench.cpp:209), one untimed warm-up call, and the median of `repeats`
    calls per block over `gsvd_blocks` distinct blocks."""
    try:
        import oracle

        if not oracle.ref_available():
            return None
    except Exception:
        return None
    info = host_cpu_info()
    cores = info["nproc"]
    spb, st, ref_out = reference_time_blocks(w, nblocks, cores)
    R = oracle.ref()
    r = R.correlation(w.x[:w.t - 1 + gsvd_blocks], w.t)
    mc = oracle.MusicCfg.make(num_sources=w.ns)

    def per_block(fn):
        return float(np.median([fn(rb) for rb in r[:gsvd_blocks]]))

    g1 = per_block(lambda rb: R.time_gsvd(w.k, rb, 0, 1, repeats))
    ga = per_block(lambda rb: R.time_gsvd(w.k, rb, 0, cores, repeats))
    s1 = per_block(lambda rb: R.time_spectrum(w.k, rb, w.h, mc, 1, repeats))
    sa = per_block(lambda rb: R.time_spectrum(w.k, rb, w.h, mc, cores, repeats))
    return {"value": 1.0 / spb, "unit": UNIT, "cores": cores, "kind": "reference", **info,
            "sample": f"{nblocks} consecutive blocks of the same {args_config_name(w)} stream through the reference "
                      f"run_locate loop (oracle/_ref = unmodified sslkit, ssl::gsvd batched float path, {cores} "
                      f"threads); stage timings: {gsvd_blocks} blocks x median of {repeats} calls after a warm-up, "
                      f"noise inverses prepared outside the timer",
            "stage_s": {"correlation": st[0], "factorization": st[1], "spectrum": st[2], "peaks": st[3]},
            "gsvd_us_per_block": 1e6 * st[1] / nblocks,
            "gsvd_1thread_us": 1e6 * g1, "gsvd_allcore_us": 1e6 * ga,
            "spectrum_1thread_us": 1e6 * s1, "spectrum_allcore_us": 1e6 * sa,
            "_ref_out": ref_out}


def args_config_name(w):
    return getattr(w, "name", "C3").upper()


def parity_in_run(w, eng_factory, ref_out, nblocks, n_fp64=3):
    """The bench scene's estimates against the reference on the same frames
    (SURVEY §8(d) parity gates): ranked direction sets vs the reference's
    production float path on every sampled block, and vs its FP64 oracle path
    (plus the broadband spectrum's relative error) on the first n_fp64."""
    import oracle

    eng = eng_factory()
    frames = w.x[:w.t - 1 + nblocks]
    out = eng.push(frames, want_power=True)
    eng.close()
    same_f = [np.array_equal(out["idx"][b][:out["count"][b]], ref_out["idx"][b][:ref_out["count"][b]])
              for b in range(nblocks)]
    R = oracle.ref()
    mc = oracle.MusicCfg.make(num_sources=w.ns)
    dbl = R.locate_frames(oracle.Workload(frames[:w.t - 1 + n_fp64], w.k, w.h, w.dirs), w.t, mc, path=2,
                          threads=os.cpu_count() or 1)
    same_d = [np.array_equal(out["idx"][b][:out["count"][b]], dbl["idx"][b][:dbl["count"][b]]) for b in range(n_fp64)]
    rel = max(float(np.max(np.abs(out["power"][b] - dbl["power"][b]) / np.abs(dbl["power"][b])))
              for b in range(n_fp64))
    return {"blocks_vs_reference_float_path": nblocks, "same_ranked_directions_float": float(np.mean(same_f)),
            "blocks_vs_reference_fp64_path": n_fp64, "same_ranked_directions_fp64": float(np.mean(same_d)),
            "pbar_max_rel_err_vs_fp64": rel}


if __name__ == "__main__":
    main()
