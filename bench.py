#!/usr/bin/env python
"""Benchmark: batched quantise + reshape-search + CSR + rANS round trip on B200.

Workload (BASELINE.json configs[1]): VGG16 split-point features, batch 256 of
(1, 256, 56, 56) post-ReLU Laplace tensors at sparsity 0.5, seeds
rank*256 .. rank*256+255, Q = 8, precision 14, N chosen by Algorithm 1 on the
device, container format v2 (FORMAT.md: W = 32 lanes, 8192-symbol blocks).

A step = compress the batch + decompress it.  Metric: GB/s of
fp32 features through encode+decode = 4*T*batch / step time, whole job.

  value  device-resident step (inputs in HBM; 822 MB per rank, larger than
         L2, so no flush is needed); timed with CUDA events on the library's
         stream, max over ranks.
  e2e    the same through the C-ABI host-buffer entry points
         (scz_compress_batch / scz_decompress_batch): pinned host features in,
         host containers out, host containers in, host features out.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: one process per GPU under torchrun; every rank codes its own 256
tensors (weak scaling, no collective on the data path; the barrier and the
max-over-ranks reduction of the timings use NCCL).
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# NVML poll period of the clock sampler (its queries share driver locks with
# the feeding thread; a coarser period keeps them off the host's critical path)
CLOCK_POLL_S = float(os.environ.get("SCZ_CLOCK_POLL_MS", "2")) / 1e3

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rANS encode+decode GB/s of fp32 features & p50 latency/tensor; bytes/element"
UNIT = "GB/s"
WORKLOADS = {
    "vgg16": dict(dims=(1, 256, 56, 56), kind="relu-laplace", sparsity=0.5, q=8,
                  name="VGG16 split-point features 1x256x56x56 post-ReLU sparsity 0.5, 8-bit"),
    "mobilenetv2": dict(dims=(1, 64, 14, 14), kind="signed", sparsity=0.0, q=8,
                        name="MobileNetV2 features[10] 1x64x14x14 signed Laplace, 8-bit"),
    "resnet50": dict(dims=(1, 512, 28, 28), kind="relu-laplace", sparsity=0.5, q=8,
                     name="ResNet-50 layer2 1x512x28x28 post-ReLU sparsity 0.5, 8-bit"),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vgg16", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=256, help="tensors per rank (weak scaling)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: this many tensors in total, shard.partition over the ranks "
                         "(config C3: 4096)")
    ap.add_argument("--format", type=int, default=2, choices=[1, 2])
    ap.add_argument("--block-syms", type=int, default=8192)
    ap.add_argument("--serialize", type=int, default=int(os.environ.get("SCZ_BENCH_SERIALIZE", "0")),
                    help="1: the rotating contexts' batch calls run in queue order (event chain)")
    ap.add_argument("--contexts", type=int, default=int(os.environ.get("SCZ_BENCH_CONTEXTS", "6")),
                    help="library contexts the device-resident steps rotate over (>= 2)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="bounded CPU-baseline sample (rank 0, N=1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip v1 / latency side measurements")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer round trip (profiling runs)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-BASELINE-config sub-records")
    return ap.parse_args()


def make_batch(wl, batch, seed0):
    from paper_2511_11664_b200.synth import make_input

    T = int(np.prod(wl["dims"]))
    out = np.empty((batch, T), np.float32)
    for i in range(batch):
        out[i] = make_input(dict(kind=wl["kind"], dims=wl["dims"], sparsity=wl["sparsity"],
                                 seed=seed0 + i))
    return out


# ------------------------------------------------------------ CPU baseline
def _cpu_worker(args):
    wl_key, seed, fmt = args
    from oracle import oracle as orc
    from paper_2511_11664_b200.synth import make_input

    wl = WORKLOADS[wl_key]
    x = make_input(dict(kind=wl["kind"], dims=wl["dims"], sparsity=wl["sparsity"], seed=seed))
    t0 = time.perf_counter()
    c = orc.compress(x, wl["dims"], wl["q"], None, 14, fmt=fmt)
    out = orc.decompress(c)
    dt = time.perf_counter() - t0
    assert out.size == x.size
    return dt, len(orc.to_bytes(c))


def cpu_baseline(wl_key, seconds, processes=None, fmt=1):
    """The oracle port (oracle/: the reference's algorithm in C + numpy) on the
    host cores: compress (with Algorithm 1) + decompress one tensor per task,
    one task per process, for ~`seconds` of wall time."""
    import multiprocessing as mp

    wl = WORKLOADS[wl_key]
    T = int(np.prod(wl["dims"]))
    cores = processes or len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    done, per_task = 0, []
    t_start = time.perf_counter()
    seed = 0
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_worker, [(wl_key, 10_000 + i, fmt) for i in range(cores)])  # warm-up
        t_start = time.perf_counter()
        while time.perf_counter() - t_start < seconds or done == 0:
            res = pool.map(_cpu_worker, [(wl_key, seed + i, fmt) for i in range(cores)])
            seed += cores
            done += len(res)
            per_task += [r[0] for r in res]
        wall = time.perf_counter() - t_start
    gbs = 4.0 * T * done / wall / 1e9
    return dict(value=gbs, unit=UNIT, cores=cores, kind="port",
                sample=f"{done} tensors of {wl['name']} (compress incl. Algorithm 1 + decompress, "
                       f"format v{fmt}) on {cores} processes, {wall:.1f} s wall; "
                       f"per-tensor p50 {statistics.median(per_task) * 1e3:.1f} ms"), per_task


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    T = int(np.prod(wl["dims"]))
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    pool = mp.get_context("fork").Pool(cores)
    seed = 0
    times, per_task = [], []
    for step in range(args.warmup + args.steps):
        tasks = [(args.workload, seed + i, 1) for i in range(cores)]
        seed += cores
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, tasks)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            per_task += [r[0] for r in res]
    pool.close()
    total = sum(times)
    value = 4.0 * T * cores * len(times) / total / 1e9
    line = dict(metric=METRIC, value=value, unit=UNIT, impl="reference", n_gpus=args.gpus,
                steps=args.steps, warmup=args.warmup, ms_per_step=1e3 * total / len(times),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64/u32",
                data="synthetic",
                config=dict(workload=wl["name"], global_batch=cores, q_bits=wl["q"],
                            format="v1 (reference wire format)", precision=14),
                cpu_baseline=dict(value=value, unit=UNIT, cores=cores, kind="port",
                                  sample=f"each step: {cores} tensors (one per host process), "
                                         "oracle C/numpy port of sczip compress+decompress; "
                                         f"per-tensor p50 {statistics.median(per_task) * 1e3:.1f} ms"),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML while the
    timed region runs: a background thread polls every ~2 ms (the timed region
    is tens of ms, too short for `nvidia-smi -lms`), and `sample()` takes one
    extra reading from the launching thread while queued work is executing."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, torch_device):
        self.nv = None
        self.samples = []
        self.stop = threading.Event()
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda._get_nvml_device_index(torch_device))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # no NVML: the line says samples=0
            self.nv = None

    def sample(self):
        if self.nv is None:
            return
        nv = self.nv
        try:
            mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
        except Exception:
            return
        self.samples.append((mhz, bits, util))

    def _poll(self):
        while not self.stop.is_set():
            self.sample()
            time.sleep(CLOCK_POLL_S)

    def __enter__(self):
        if self.nv is not None:
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.thread.join(timeout=5)

    def summary(self):
        if not self.samples:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=[], samples=0)
        reasons = set()
        for _, bits, _ in self.samples:
            for name, attr in self.REASONS:
                if bits & getattr(self.nv, attr, 0):
                    reasons.add(name)
        loaded = [m for m, _, u in self.samples if u > 0] or [m for m, _, _ in self.samples]
        return dict(sm_mhz=statistics.median(loaded), sm_max_mhz=self.max_mhz, reasons=sorted(reasons),
                    samples=len(self.samples), samples_under_load=sum(1 for s in self.samples if s[2] > 0),
                    source=f"NVML, polled every ~{CLOCK_POLL_S * 1e3:.0f} ms during the timed region",
                    note="samples_under_load counts NVML utilization > 0, a trailing average over >= 1/6 s: "
                         "a timed region of ~0.1 s after an idle phase can read 0 while every sample "
                         "was taken with the GPU busy")


def gpu_local_cpus(torch, device):
    """CPUs NVML reports as local to `device` (empty set if unknown)."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda._get_nvml_device_index(device))
        n = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        return {i for i in range(n) if (words[i // 64] >> (i % 64)) & 1}
    except Exception:
        return set()


# -------------------------------------------------------------- our arm
# What bounds the rANS kernels below the HBM roofline (ncu --set full,
# profiles/r2h/ncu_full_summary.txt and DESIGN.md 'Where the step time goes').
LIMITERS = {
    "k_rans_dec_v2": "not HBM: instruction issue (~73 % active, ~41 warp instructions per 32-symbol step) and "
                     "shared-memory wavefronts (two random slot-table lookups per step, ~1.9x the conflict-free "
                     "count); residency is capped at 32 warps/SM by the 80 KB table per CTA",
    "k_rans_enc_v2": "not HBM: instruction issue (~73 % active, ~25 instructions per lane-step: renormalisation "
                     "tests, ballot-scan byte placement, exact-reciprocal state update)",
}


def algorithmic_bytes(name, infos, T, nblk_bytes):
    """Bytes a kernel must move per launch, batch-summed."""
    nnz = sum(int(i["nnz"]) for i in infos)
    N = sum(int(i["n_rows"]) for i in infos)
    S = sum(int(i["payload_len"]) for i in infos)
    B = len(infos)
    w = max(int(i["sym_bytes"]) for i in infos)
    L = 2 * nnz + N
    name = name.split("/")[0]  # width variants share the formula
    return {
        "k_stats": 4 * T * B + T * B // 8,
        "k_quantize": 4 * T * B + T * B // 8 + nnz,
        "k_colhist": T * B // 8,
        "k_materialize": T * B // 8 + (nnz + N) * w,
        "k_rans_enc_v2": nnz + (nnz + N) * w + S,
        "k_rans_enc_v1": nnz + (nnz + N) * w + S,
        "k_pack": 2 * S,
        "k_rans_dec_v2": S + L * w,
        "k_rans_dec_v1": S + L * w,
        "k_row_sums": N * w,
        "k_rows_out": L * w + 4 * T * B,
    }.get(name)


def run_ours(args):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SCZ_BENCH_DEVICE pins every rank to one GPU (a multi-rank dry run of the
    # torchrun path on a one-GPU box); NCCL refuses two ranks on one device,
    # so that mode uses gloo for the barrier and the reductions
    dev_override = os.environ.get("SCZ_BENCH_DEVICE")
    if dev_override is not None:
        local = int(dev_override)
    torch.cuda.set_device(local)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("SCZ_BENCH_DIST_BACKEND", "gloo" if dev_override is not None else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    red_dev = torch.device("cuda", local) if backend == "nccl" else None

    from paper_2511_11664_b200 import _native, shard

    # Host threads (and the pinned buffers they touch first) on the GPU's own
    # NUMA node: the e2e path is PCIe-bound, and DMA to far-socket memory
    # crosses the inter-socket link.  The CPU baseline gets all cores back.
    all_cpus = os.sched_getaffinity(0)
    near = gpu_local_cpus(torch, local) & all_cpus
    if near:
        os.sched_setaffinity(0, near)

    wl = WORKLOADS[args.workload]
    T = int(np.prod(wl["dims"]))
    # the tensors this rank codes: its own `batch` seeds (weak scaling,
    # shard.weak_seeds) or its contiguous slice of --global-batch (strong
    # scaling, shard.partition); tensors are independent, no data collective
    if args.global_batch:
        lo, hi = shard.partition(args.global_batch, world, rank)
        seeds = range(lo, hi)
        scaling = "strong"
    else:
        seeds = shard.weak_seeds(args.batch, rank)
        scaling = "weak"
    B = len(seeds)
    total_units = args.global_batch if args.global_batch else args.batch * world
    ctx = _native.context(local)
    lib = ctx.lib
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    host = torch.empty((B, T), dtype=torch.float32).pin_memory()
    host.numpy()[:] = make_batch(wl, B, seeds.start)
    x_dev = host.cuda(local)
    out_dev = torch.empty_like(x_dev)
    torch.cuda.synchronize()

    batch = _native.Batch()
    h_info = (_native.Info * B)()

    def device_step(fmt=args.format):
        ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x_dev.data_ptr()), T, B, wl["q"], -1, 14,
                                       fmt, 32, args.block_syms, ctypes.byref(batch)))
        ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), h_info))
        ctx.check(lib.scz_decode_batch_async(ctx.h, h_info, B, ctypes.c_void_p(batch.d_freqs),
                                             ctypes.c_void_p(batch.d_block_bytes),
                                             ctypes.c_void_p(batch.d_payload),
                                             ctypes.c_void_p(out_dev.data_ptr())))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        return shard.reduce_max(v, dist, red_dev)

    # ---- device-resident timed region -------------------------------------
    # Library contexts (own stream + scratch each; --contexts, default 6)
    # rotate between steps: step i + 2's encode is queued before the host
    # reads step i's headers (scz_batch_sync) and queues its decode, so the
    # GPU never idles on the host round trip.  Every step still compresses and decompresses
    # the whole batch; the timing is CUDA events on both streams.
    # (scz_decode_batch_device avoids the host round trip altogether, but
    # without the headers it must launch every symbol-class / K variant the
    # plan allows; with the chosen variants known on the host this path is
    # faster for a full batch.)
    # (each context holds a whole batch of scratch, about 6x the fp32 input:
    # large per-rank batches rotate over fewer contexts)
    NC = max(2, args.contexts if 4 * T * B <= (2 << 30) else min(args.contexts, 3))
    ctxs = [ctx] + [_native.Context(local) for _ in range(NC - 1)]
    streams = [stream] + [torch.cuda.ExternalStream(c.stream, device=torch.device("cuda", local))
                          for c in ctxs[1:]]
    batches = [_native.Batch() for _ in range(NC)]
    infos = [(_native.Info * B)() for _ in range(NC)]
    outs = [out_dev] + [torch.empty_like(x_dev) for _ in range(NC - 1)]

    # --serialize 1: every queued batch call waits for the one
    # queued before it (an event chain across the context streams), so the
    # device runs the steps' kernels in queue order instead of interleaving
    # kernels of several contexts; the header read-back of a step still waits
    # only for that step's encode.
    chain_ev = [None]

    def chain(k):
        if args.serialize and chain_ev[0] is not None:
            streams[k].wait_event(chain_ev[0])

    def mark(k):
        if args.serialize:
            e = torch.cuda.Event()
            e.record(streams[k])
            chain_ev[0] = e

    def enc(k, fmt=None):
        c = ctxs[k]
        chain(k)
        c.check(lib.scz_encode_batch(c.h, ctypes.c_void_p(x_dev.data_ptr()), T, B, wl["q"], -1, 14,
                                     fmt or args.format, 32, args.block_syms, ctypes.byref(batches[k])))
        mark(k)

    def dec(k):
        c = ctxs[k]
        c.check(lib.scz_batch_sync(c.h, ctypes.byref(batches[k]), infos[k]))
        chain(k)
        c.check(lib.scz_decode_batch_async(c.h, infos[k], B, ctypes.c_void_p(batches[k].d_freqs),
                                           ctypes.c_void_p(batches[k].d_block_bytes),
                                           ctypes.c_void_p(batches[k].d_payload),
                                           ctypes.c_void_p(outs[k].data_ptr())))
        mark(k)

    host_ms = []  # host time spent queueing each step (diagnostic)
    step_ev = []  # (stream, event) after each step's decode (diagnostic)

    def pipelined(n, clocks=None, record=False, fmt=None):
        # step i's encode is queued NC - 1 steps ahead of its decode
        for i in range(min(NC - 1, n)):
            enc(i % NC, fmt)
        for i in range(n):
            t0 = time.perf_counter()
            if i + NC - 1 < n:
                enc((i + NC - 1) % NC, fmt)
            dec(i % NC)
            if record:
                host_ms.append((time.perf_counter() - t0) * 1e3)
                e = torch.cuda.Event(enable_timing=True)
                e.record(streams[i % NC])
                step_ev.append(e)
            if clocks:
                clocks.sample()

    # a context's launch sequence runs eagerly on first sight, is captured
    # into a CUDA graph on the second and replayed from then on: three rounds
    # so the timed region only replays
    for _ in range(max(3, args.warmup)):
        pipelined(NC)
    for _ in range(args.warmup):
        device_step()
    barrier()
    l0 = sum(c.launches for c in ctxs)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(NC)]
    clocks = ClockSampler(local)
    gc.collect()
    gc.disable()  # no collector pause while the host feeds the queue
    with clocks:
        barrier()
        ev0.record(streams[0])
        for st_ in streams[1:]:
            st_.wait_event(ev0)
        pipelined(args.steps, None, record=True)  # clocks: the poll thread only (NVML off the feeding thread)
        for k in range(NC):
            ev_end[k].record(streams[k])
        barrier()
    gc.enable()
    launches = sum(c.launches for c in ctxs) - l0
    # per-step completion gaps on the device (decode-end to decode-end)
    done = [ev0.elapsed_time(e) for e in step_ev]
    gaps = sorted(b - a for a, b in zip(done, done[1:])) or [0.0]
    step_diag = dict(host_queue_ms_p50=statistics.median(host_ms), host_queue_ms_max=max(host_ms),
                     step_gap_ms_p50=statistics.median(gaps), step_gap_ms_max=gaps[-1])
    ms = max(ev0.elapsed_time(e) for e in ev_end) / args.steps
    ms = max_over_ranks(ms)
    value = 4.0 * T * total_units / (ms * 1e-3) / 1e9

    statuses = (ctypes.c_int32 * B)()
    for k in range(NC):
        ctxs[k].check(lib.scz_decode_status(ctxs[k].h, B, statuses))
        assert all(v == 0 for v in statuses), "decode status"

    # ---- v1 (the reference's wire format) through the same pipeline --------
    # One serial rANS chain per tensor: a batch costs one chain's latency, so
    # the contexts' batches in flight (encodes queued NC - 1 steps ahead of
    # their decodes) are what fill the GPU's schedulers.
    v1_pipe = None
    if not args.no_extras and rank == 0 and args.format == 2:
        for _ in range(3):  # eager, graph capture, replay: per context
            pipelined(NC, fmt=1)
        torch.cuda.synchronize()
        n1 = 2 * NC
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(NC)]
        e0.record(streams[0])
        for st_ in streams[1:]:
            st_.wait_event(e0)
        pipelined(n1, fmt=1)
        for k in range(NC):
            e1[k].record(streams[k])
        torch.cuda.synchronize()
        ms1 = max(e0.elapsed_time(e) for e in e1) / n1
        for k in range(NC):
            ctxs[k].check(lib.scz_decode_status(ctxs[k].h, B, statuses))
            assert all(v == 0 for v in statuses), "v1 decode status"
        assert torch.equal(outs[0], outs[1]), "v1 reconstructions differ between contexts"
        v1_pipe = dict(value=4.0 * T * B / (ms1 * 1e-3) / 1e9, unit=UNIT, ms_per_step=ms1, steps=n1,
                       contexts=NC, batch=B,
                       schedule=f"{NC} contexts, encodes queued {NC - 1} steps ahead of their decodes "
                                "(as the headline value)")

    # ---- per-kernel times (separate pass: per-launch events, no graphs) ----
    ctx.set_timing(True)
    ctx.read_timing()
    for _ in range(3):
        device_step()
    torch.cuda.synchronize()
    kt = ctx.read_timing()
    ctx.set_timing(False)
    device_step()  # outputs of the default context for the checks below
    torch.cuda.synchronize()
    kt_steps = 3
    assert torch.equal(outs[1], out_dev), "second context's reconstruction differs"

    status = (ctypes.c_int32 * B)()
    ctx.check(lib.scz_decode_status(ctx.h, B, status))
    infos = [{f: getattr(h_info[i], f) for f, _ in _native.Info._fields_} for i in range(B)]
    assert all(s == 0 for s in status) and all(i["status"] == 0 for i in infos), "device status"
    # every reconstruction within the quantisation bound, zeros exact (tensor.py:143-156)
    scales = torch.tensor([i["scale"] for i in infos], device=x_dev.device, dtype=torch.float32)
    err = (out_dev - x_dev).abs().amax(dim=1)
    assert bool((err <= scales * 1.0001 + 1e-6).all()), "reconstruction outside the quantisation bound"
    assert bool((out_dev[x_dev == 0] == 0).all())
    total_bytes = sum(i["payload_len"] + 60 + 4 * len(wl["dims"]) + 2 * i["alphabet"] +
                      (12 + 4 * i["n_blocks"] if args.format == 2 else 0) for i in infos)
    bpe = total_bytes / (T * B)

    # ---- roofline of the dominant kernel ----------------------------------
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    dom = max(kt.items(), key=lambda kv: kv[1][0]) if kt else None
    roofline = None
    kernel_share = {}
    if dom:
        step_ms_sum = sum(v[0] for v in kt.values())
        kernel_share = {k: round(v[0] / step_ms_sum, 4) for k, v in sorted(kt.items(), key=lambda kv: -kv[1][0])}
        name, (tot_ms, n) = dom
        per_launch_ms = tot_ms / n
        launches_per_step = n / kt_steps
        ab = algorithmic_bytes(name, infos, T, None)
        achieved = (ab / launches_per_step) / (per_launch_ms * 1e-3) / 1e9 if ab else None
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            traffic = json.load(open(prof)).get(name)
        roofline = dict(kernel=name, bound="hbm", achieved=achieved, peak=peak, unit="GB/s",
                        frac=(achieved / peak) if achieved else None, traffic=traffic,
                        algorithmic_bytes_per_launch=(ab / launches_per_step) if ab else None,
                        launch_ms=per_launch_ms, peak_source=peak_src)
        if name.split("/")[0] in LIMITERS:
            roofline["limiter"] = LIMITERS[name.split("/")[0]]
    pipe_bytes = 8 * T * B + 2 * total_bytes
    pipeline_roofline = dict(achieved=pipe_bytes / (ms * 1e-3) / 1e9, peak=peak, unit="GB/s",
                             frac=pipe_bytes / (ms * 1e-3) / 1e9 / peak,
                             bytes_per_step="8*T*batch + 2*container bytes")

    # ---- e2e through the host-buffer C-ABI ---------------------------------
    # A round trip per step: pinned host features -> scz_compress_batch ->
    # host containers -> scz_decompress_batch -> pinned host features.  The
    # two calls run as a two-stage pipeline (one host thread each, separate
    # contexts and streams) so step i's decompress overlaps step i + 1's
    # compress: PCIe carries H2D and D2H traffic at the same time.  Two
    # compress contexts alternate so a step's containers stay intact until
    # its decompress has consumed them (three slots: compress may run up to
    # two steps ahead, which keeps both PCIe directions busy).
    e2e = None
    if not args.no_e2e:
        e2e_ms, io, h_out, e2e_status = run_e2e(args, torch, _native, lib, local, host, T, B, wl, pairs=E2E_PAIRS)
        e2e_ms = max_over_ranks(e2e_ms)
        e2e_value = 4.0 * T * total_units / (e2e_ms * 1e-3) / 1e9
        assert all(s == 0 for s in e2e_status)
        assert torch.equal(h_out, out_dev.cpu()), "host-path reconstruction differs from device path"
        e2e = dict(value=e2e_value, unit=UNIT, h2d_bytes_per_step=io["h2d"],
                   d2h_bytes_per_step=io["d2h"], ms_per_step=e2e_ms, stage_ms=io["stage_ms"],
                   path="scz_compress_batch + scz_decompress_batch, pinned host buffers",
                   schedule=f"{E2E_PAIRS} x 2-stage pipeline: decompress(step i) || compress(step i+1)",
                   timing="host clock between decompress completions in steady state",
                   host_cpus=f"{len(near)} GPU-local CPUs (NVML affinity)" if near else "unrestricted")

    extras = {}
    if not args.no_extras and rank == 0:
        extras = side_measurements(args, ctx, lib, wl, T, x_dev, out_dev, stream, torch)
        if v1_pipe and "v1_reference_format" in extras:
            v1 = extras["v1_reference_format"]
            seq = dict(value=v1.pop("value"), ms_per_step=v1.pop("ms_per_step"),
                       schedule="one context: encode, header read, decode")
            extras["v1_reference_format"] = dict(v1_pipe, sequential=seq, **v1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.sched_setaffinity(0, all_cpus)
        cpu, _ = cpu_baseline(args.workload, args.cpu_seconds)

    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps,
            warmup=args.warmup, ms_per_step=ms, higher_is_better=True, scaling=scaling,
            vs_baseline=None, dtype="u8/u32 (fp32 in/out, fp64 quant params)", data="synthetic",
            config=dict(workload=wl["name"], global_batch=total_units, per_gpu_batch=B, q_bits=wl["q"],
                        precision=14, format=f"v{args.format}", lanes=32,
                        block_syms=args.block_syms, reshape="Algorithm 1 on device",
                        parallelism=f"dp{world} (independent tensors, no collective)",
                        l2=f"inputs {4 * T * B / 1e6:.0f} MB per rank "
                           + ("> 126 MB L2 (no flush needed)" if 4 * T * B > 126e6 else
                              "< 126 MB L2: NOT flushed between steps")),
            bytes_per_element=bpe,
            e2e=e2e,
            roofline=roofline, pipeline_roofline=pipeline_roofline, kernel_share=kernel_share,
            gpu_launches=launches, clocks=clocks.summary(), step_diagnostics=step_diag, cpu_baseline=cpu, **extras)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


E2E_SLOTS = int(os.environ.get("SCZ_E2E_SLOTS", "3"))
V1_E2E_PAIRS = int(os.environ.get("SCZ_V1_E2E_PAIRS", "1"))
E2E_PAIRS = int(os.environ.get("SCZ_E2E_PAIRS", "1"))


def run_e2e(args, torch, _native, lib, device, host, T, B, wl, pairs=1):
    """Pipelined round trips through the host-buffer entry points; returns
    (ms per step, bytes per step, last output, last status).  `pairs`
    compressor/decompressor thread pairs each run the two-stage pipeline over
    every pairs-th step (v1: one serial chain per tensor, so more batches in
    flight fill the GPU)."""
    import threading

    ns = E2E_SLOTS
    nsl = ns * pairs
    cctx = [_native.Context(device) for _ in range(nsl)]  # compress slots
    dctx = [_native.Context(device) for _ in range(pairs)]
    slot = [dict(infos=ctypes.POINTER(_native.Info)(), pay=ctypes.POINTER(ctypes.c_uint8)(),
                 fr=ctypes.POINTER(ctypes.c_uint32)(), bl=ctypes.POINTER(ctypes.c_uint32)(),
                 sizes=(ctypes.c_uint64 * 3)()) for _ in range(nsl)]
    free = [threading.Semaphore(1) for _ in range(nsl)]
    ready = [threading.Semaphore(0) for _ in range(nsl)]
    h_out = torch.empty((B, T), dtype=torch.float32).pin_memory()
    status = [(ctypes.c_int32 * B)() for _ in range(pairs)]
    # every compress slot and the decompress context see their shapes twice
    # (eager, then graph capture) before the timed window opens
    n_warm = pairs * max(args.warmup, 2 * ns + 1)
    n_total = n_warm + args.steps
    done_at = [0.0] * n_total
    c_ms, d_ms = [], []
    errors = []
    io = {}

    def compressor(t):
        try:
            for i in range(t, n_total, pairs):
                k = i % nsl
                free[k].acquire()
                sl, c = slot[k], cctx[k]
                t0 = time.perf_counter()
                c.check(lib.scz_compress_batch(c.h, ctypes.c_void_p(host.data_ptr()), T, B, wl["q"], -1, 14,
                                               args.format, 32, args.block_syms, ctypes.byref(sl["infos"]),
                                               ctypes.byref(sl["pay"]), ctypes.byref(sl["fr"]),
                                               ctypes.byref(sl["bl"]), sl["sizes"]))
                c_ms.append((time.perf_counter() - t0) * 1e3)
                ready[k].release()
        except Exception as e:  # surfaced by the main thread
            errors.append(e)
            for r in ready:
                r.release()

    def decompressor(t):
        try:
            dc = dctx[t]
            for i in range(t, n_total, pairs):
                k = i % nsl
                ready[k].acquire()
                if errors:
                    return
                sl = slot[k]
                z = sl["sizes"]
                t0 = time.perf_counter()
                dc.check(lib.scz_decompress_batch(dc.h, sl["infos"], B, sl["fr"], z[1], sl["bl"], z[2],
                                                  sl["pay"], z[0], ctypes.c_void_p(h_out.data_ptr()), status[t]))
                done_at[i] = time.perf_counter()
                d_ms.append((done_at[i] - t0) * 1e3)
                io["h2d"] = 4 * T * B + z[0] + 4 * z[1] + 4 * z[2]
                io["d2h"] = B * ctypes.sizeof(_native.Info) + z[0] + 4 * z[1] + 4 * z[2] + 4 * T * B + 4 * B
                free[k].release()
        except Exception as e:
            errors.append(e)
            for f in free:
                f.release()

    th = [threading.Thread(target=f, args=(t,)) for t in range(pairs) for f in (compressor, decompressor)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    w = n_warm
    # steady state: completions per unit time, from the w-th completion to
    # the last (pairs > 1 completes steps slightly out of order)
    t_done = sorted(done_at)
    ms = (t_done[-1] - t_done[w - 1]) * 1e3 / args.steps
    io["stage_ms"] = dict(compress=statistics.median(c_ms[w:]), decompress=statistics.median(d_ms[w:]))
    return ms, io, h_out, [v for st in status for v in st]


def side_measurements(args, ctx, lib, wl, T, x_dev, out_dev, stream, torch):
    """Per-tensor p50 latency (B = 1, device resident) and the v1 (reference
    wire format) batch throughput."""
    from paper_2511_11664_b200 import _native

    res = {}
    batch = _native.Batch()
    info1 = (_native.Info * 1)()
    x0 = ctypes.c_void_p(x_dev[0].data_ptr())
    o0 = ctypes.c_void_p(out_dev[0].data_ptr())
    lat_enc, lat_dec = [], []

    # L2 flush between repetitions: a 256 MB buffer (> 126 MB L2) is written
    # once and READ before every repetition -- reading evicts the tensor's
    # lines without leaving 256 MB of dirty lines whose write-back would then
    # compete with the timed kernels
    flush_buf = torch.ones(64 << 20, dtype=torch.float32, device=x_dev.device)
    flush_sink = torch.empty((), dtype=torch.float32, device=x_dev.device)

    def flush():
        with torch.cuda.stream(stream):
            torch.sum(flush_buf, dim=0, out=flush_sink)

    def one(timed, bs=args.block_syms):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        flush()  # the tensor (3.2 MB) would otherwise stay in L2 between repetitions
        a.record(stream)
        ctx.check(lib.scz_encode_batch(ctx.h, x0, T, 1, wl["q"], -1, 14, 2, 32, bs,
                                       ctypes.byref(batch)))
        ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info1))
        b.record(stream)
        ctx.check(lib.scz_decode_batch_async(ctx.h, info1, 1, ctypes.c_void_p(batch.d_freqs),
                                             ctypes.c_void_p(batch.d_block_bytes),
                                             ctypes.c_void_p(batch.d_payload), o0))
        c.record(stream)
        c.synchronize()
        if timed:
            lat_enc.append(a.elapsed_time(b) * 1e3)
            lat_dec.append(b.elapsed_time(c) * 1e3)

    # latency: the production path (repeated shapes replay captured CUDA graphs)
    for it in range(50):
        one(it >= 10)
    # the device round trip: decode straight from the encoder's on-device
    # headers (scz_decode_batch_device), no host read of the headers between
    lat_dev = []
    for it in range(50):
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush()
        a.record(stream)
        ctx.check(lib.scz_encode_batch(ctx.h, x0, T, 1, wl["q"], -1, 14, 2, 32, args.block_syms,
                                       ctypes.byref(batch)))
        ctx.check(lib.scz_decode_batch_device(ctx.h, o0))
        c.record(stream)
        c.synchronize()
        if it >= 10:
            lat_dev.append(a.elapsed_time(c) * 1e3)
    st1 = (ctypes.c_int32 * 1)()
    ctx.check(lib.scz_decode_status(ctx.h, 1, st1))
    assert st1[0] == 0
    # per-kernel breakdown: a separate pass with per-launch events (eager)
    ctx.set_timing(True)
    for it in range(15):
        if it == 5:
            ctx.read_timing()
        one(False)
    kt = ctx.read_timing()
    ctx.set_timing(False)
    res["latency_us_p50"] = dict(
        encode=statistics.median(lat_enc), decode=statistics.median(lat_dec),
        encode_plus_decode=statistics.median([e + d for e, d in zip(lat_enc, lat_dec)]),
        device_round_trip=statistics.median(lat_dev),
        tensor=str(wl["dims"]), format="v2",
        note="device-resident, L2 flushed before every repetition; encode includes the header D2H sync "
             "(scz_batch_sync); device_round_trip = scz_encode_batch + scz_decode_batch_device (headers stay "
             "on the device); kernel_us from a separate per-launch-event pass",
        kernel_us={k: round(1e3 * ms / n, 2) for k, (ms, n) in sorted(kt.items(), key=lambda kv: -kv[1][0])})
    # the block-size trade-off: shorter v2 blocks shorten the serial rANS
    # chains (more blocks in flight for one tensor) at the cost of 128 state
    # bytes + 4 table bytes per block
    trade = []
    for bs in (4096, 2048):
        lat_enc.clear()
        lat_dec.clear()
        for it in range(40):
            one(it >= 10, bs)
        size = info1[0].payload_len + 60 + 4 * len(wl["dims"]) + 2 * info1[0].alphabet + 12 + 4 * info1[0].n_blocks
        trade.append(dict(block_syms=bs, encode_plus_decode_us=statistics.median(
            [e + d for e, d in zip(lat_enc, lat_dec)]), bytes_per_element=size / T))
    res["latency_us_p50"]["block_size_tradeoff"] = trade
    # v1: the reference's single-stream format, one warp per tensor
    B = x_dev.shape[0]
    h_info = (_native.Info * B)()
    for it in range(3):
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x_dev.data_ptr()), T, B, wl["q"], -1, 14,
                                       1, 32, args.block_syms, ctypes.byref(batch)))
        ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), h_info))
        ctx.check(lib.scz_decode_batch_async(ctx.h, h_info, B, ctypes.c_void_p(batch.d_freqs),
                                             ctypes.c_void_p(batch.d_block_bytes),
                                             ctypes.c_void_p(batch.d_payload),
                                             ctypes.c_void_p(out_dev.data_ptr())))
        c.record(stream)
        c.synchronize()
    v1_ms = a.elapsed_time(c)
    res["v1_reference_format"] = dict(value=4.0 * T * B / (v1_ms * 1e-3) / 1e9, unit=UNIT,
                                      ms_per_step=v1_ms, batch=B,
                                      note="bit-exact reference wire format; serial stream per tensor")
    # v1 end to end (like-for-like with the reference arm's format): the same
    # pipelined host-buffer round trip as `e2e`, format 1
    if not args.no_e2e:
        import copy
        a1 = copy.copy(args)
        a1.format, a1.steps, a1.warmup = 1, 5, 0
        host = x_dev.cpu().pin_memory()
        a1.steps = 12
        e_ms, io, h_out, st1 = run_e2e(a1, torch, _native, lib, x_dev.device.index or 0, host, T, B, wl,
                                       pairs=V1_E2E_PAIRS)
        assert all(v == 0 for v in st1)
        res["v1_reference_format"]["e2e"] = dict(
            value=4.0 * T * B / (e_ms * 1e-3) / 1e9, unit=UNIT, ms_per_step=e_ms, steps=a1.steps,
            h2d_bytes_per_step=io["h2d"], d2h_bytes_per_step=io["d2h"],
            path="scz_compress_batch + scz_decompress_batch (format 1), pinned host buffers",
            schedule=f"{V1_E2E_PAIRS} compress/decompress thread pairs, each a 2-stage pipeline")
    if not args.no_configs:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peak = float(json.load(open(peaks_path))["hbm_gbs"]) if os.path.exists(peaks_path) else 6650.0
        t0 = time.perf_counter()
        res["configs"] = config_records(args, torch, _native, x_dev.device.index or 0, peak)
        res["configs"]["wall_s"] = round(time.perf_counter() - t0, 1)
        c2 = res["configs"].get("C2-vgg16-batch256", {}).get("v2")
        if c2:  # SURVEY 8d's encode-side target, surfaced from the C2 record
            res["encode_decode_roofline"] = dict(
                encode=c2["encode_roofline"], decode=c2["decode_roofline"], encode_ms=c2["encode_ms"],
                decode_ms=c2["decode_ms"], peak_gbs=peak,
                note="encode-only / decode-only device time of the 256-tensor VGG16 batch (CUDA events, one "
                     "context, not pipelined); algorithmic bytes 4T + S per tensor")
    return res


# ------------------------------------------------ every BASELINE config
CONTAINER_FIXED = 4 + 4 + 8 + 4 + 4 + 8 + 8 + 8 + 4 + 8  # container.py:62 without dims / freqs


def container_bytes(info, ndims):
    """Total .scz bytes of one tensor (container.py:62; FORMAT.md v2 adds 12 + 4 n_blocks)."""
    b = CONTAINER_FIXED + 4 * ndims + 2 * int(info.alphabet) + int(info.payload_len)
    if int(info.version) == 2:
        b += 12 + 4 * int(info.n_blocks)
    return b


class DeviceBatch:
    """Encode / decode of one device-resident batch through the C ABI on one
    library context, timed with CUDA events on the context's stream:
    encode = scz_encode_batch, decode = scz_decode_batch_async (after the
    host read the headers with scz_batch_sync).  Optionally reads a 256 MB
    buffer on the same stream before every timed repetition (L2 flush) when
    the batch is smaller than the 126 MB L2."""

    def __init__(self, torch, _native, device):
        self.torch = torch
        self.ctx = _native.Context(device)
        self.lib = self.ctx.lib
        self.native = _native
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=torch.device("cuda", device))
        self.flush_buf = torch.ones(64 << 20, dtype=torch.float32, device=torch.device("cuda", device))
        self.flush_sink = torch.empty((), dtype=torch.float32, device=torch.device("cuda", device))
        self.batch = _native.Batch()

    def flush(self):  # read 256 MB (> L2): evicts the batch without leaving dirty lines
        with self.torch.cuda.stream(self.stream):
            self.torch.sum(self.flush_buf, dim=0, out=self.flush_sink)

    def run(self, x, out, B, T, q, fmt, bs, n_rows=-1, reps=5, warm=3, flush=False):
        """[(encode ms, decode ms)] of `reps` timed repetitions + the infos."""
        torch, lib, c = self.torch, self.lib, self.ctx
        infos = (self.native.Info * B)()
        st = (ctypes.c_int32 * B)()
        res = []
        for r in range(warm + reps):  # eager, graph capture, replay, then timed replays
            if flush:
                self.flush()
            e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            e0.record(self.stream)
            c.check(lib.scz_encode_batch(c.h, ctypes.c_void_p(x.data_ptr()), T, B, q, n_rows, 14, fmt, 32, bs,
                                         ctypes.byref(self.batch)))
            e1.record(self.stream)
            c.check(lib.scz_batch_sync(c.h, ctypes.byref(self.batch), infos))
            e2.record(self.stream)
            c.check(lib.scz_decode_batch_async(c.h, infos, B, ctypes.c_void_p(self.batch.d_freqs),
                                               ctypes.c_void_p(self.batch.d_block_bytes),
                                               ctypes.c_void_p(self.batch.d_payload),
                                               ctypes.c_void_p(out.data_ptr())))
            e3.record(self.stream)
            c.check(lib.scz_decode_status(c.h, B, st))
            assert all(v == 0 for v in st) and all(infos[i].status == 0 for i in range(B)), "device status"
            if r >= warm:
                res.append((e0.elapsed_time(e1), e2.elapsed_time(e3)))
        return res, infos


def config_records(args, torch, _native, device, peak):
    """One record per BASELINE.json config on this GPU: device
    encode / decode times (CUDA events), throughput, p50 latency, bytes per
    element in both formats, encode / decode roofline fractions, and the
    oracle port (the reference algorithm in C + numpy) timed beside it on one
    host core for a bounded sample."""
    from oracle import oracle as orc
    from paper_2511_11664_b200.synth import make_input

    dev = DeviceBatch(torch, _native, device)
    recs = {}

    def dev_tensor(specs):
        xs = np.stack([make_input(sp) for sp in specs])
        return torch.from_numpy(xs).to(torch.device("cuda", device))

    def summarize(name, xs, dims, q, fmt, bs, reps, flush, n_rows=-1):
        B, T = xs.shape
        out = torch.empty_like(xs)
        times, infos = dev.run(xs, out, B, T, q, fmt, bs, n_rows, reps=reps, flush=flush)
        enc = statistics.median(t[0] for t in times)
        dec = statistics.median(t[1] for t in times)
        sbytes = sum(container_bytes(infos[i], len(dims)) for i in range(B))
        err = (out - xs).abs().amax(dim=1)
        scales = torch.tensor([infos[i].scale for i in range(B)], device=xs.device, dtype=torch.float32)
        assert bool((err <= scales * 1.0001 + 1e-6).all()), name
        r = dict(format=f"v{fmt}", batch=B, encode_ms=enc, decode_ms=dec, gbs=4.0 * T * B / ((enc + dec) * 1e-3) / 1e9,
                 bytes_per_element=sbytes / (T * B),
                 encode_roofline=(4.0 * T * B + sbytes) / (enc * 1e-3) / 1e9 / peak,
                 decode_roofline=(4.0 * T * B + sbytes) / (dec * 1e-3) / 1e9 / peak,
                 n_rows=int(infos[0].n_rows), n_cols=int(infos[0].n_cols))
        if fmt == 2:
            r["block_syms"] = bs
        return r, infos

    def cpu_p50(spec, q, n=3):
        x = make_input(spec)
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            c = orc.compress(x, spec["dims"], q, None, 14)
            orc.decompress(c)
            ts.append((time.perf_counter() - t0) * 1e3)
        return dict(ms_p50=statistics.median(ts), cores=1, kind="port",
                    sample=f"{n} x compress (Algorithm 1) + decompress of the same tensor, v1, one process")

    # C1: one ResNet-50 layer2 tensor, sparsity 0.5 (primary) and 0.9 (the reference's test value)
    for sp in (0.5, 0.9):
        spec = dict(kind="relu-laplace", dims=(1, 512, 28, 28), sparsity=sp, seed=42)
        x = dev_tensor([spec])
        v2, _ = summarize("C1", x, spec["dims"], 8, 2, args.block_syms, 30, True)
        v1, _ = summarize("C1v1", x, spec["dims"], 8, 1, args.block_syms, 3, True)
        recs[f"C1-resnet50-layer2-relu{sp}"] = dict(
            tensor="(1, 512, 28, 28)", v2=dict(v2, latency_us_p50=1e3 * (v2["encode_ms"] + v2["decode_ms"])),
            v1=dict(v1, latency_us_p50=1e3 * (v1["encode_ms"] + v1["decode_ms"])),
            cpu_baseline=cpu_p50(spec, 8), l2="single tensor: 256 MB L2 flush before every repetition")
    # C2: VGG16 batch 256 (serial encode / decode rooflines; the headline is the pipelined value)
    wl = WORKLOADS["vgg16"]
    x = dev_tensor([dict(kind=wl["kind"], dims=wl["dims"], sparsity=wl["sparsity"], seed=i) for i in range(256)])
    v2, _ = summarize("C2vgg", x, wl["dims"], 8, 2, args.block_syms, 3, False)
    v1, _ = summarize("C2vgg1", x, wl["dims"], 8, 1, args.block_syms, 1, False)
    recs["C2-vgg16-batch256"] = dict(v2=v2, v1=v1, note="one context, encode then decode (not pipelined)")
    del x
    # C2: MobileNetV2 features[10], signed (z = 131), batch 256: 12.8 MB < L2, flushed
    spec = [dict(kind="signed", dims=(1, 64, 14, 14), seed=i) for i in range(256)]
    x = dev_tensor(spec)
    v2, _ = summarize("C2mnv2", x, (1, 64, 14, 14), 8, 2, args.block_syms, 5, True)
    v1, _ = summarize("C2mnv2v1", x, (1, 64, 14, 14), 8, 1, args.block_syms, 3, True)
    lat, _ = summarize("C2mnv2lat", x[:1].contiguous(), (1, 64, 14, 14), 8, 2, args.block_syms, 30, True)
    recs["C2-mobilenetv2-batch256"] = dict(v2=v2, v1=v1, latency_us_p50=1e3 * (lat["encode_ms"] + lat["decode_ms"]),
                                           cpu_baseline=cpu_p50(spec[0], 8, 5),
                                           l2="batch 12.8 MB < L2: 256 MB flush before every repetition")
    del x
    # C3: ResNet-50 features, batch 4096 on this GPU (seeds 0..511, each tensor 8 times: host generation time)
    spec = [dict(kind="relu-laplace", dims=(1, 512, 28, 28), sparsity=0.5, seed=i) for i in range(512)]
    x1 = dev_tensor(spec)
    x = x1.repeat(8, 1)
    del x1
    v2, _ = summarize("C3", x, (1, 512, 28, 28), 8, 2, args.block_syms, 2, False)
    recs["C3-resnet50-batch4096"] = dict(v2=v2, note="N = 1; bench.py --workload resnet50 --global-batch 4096 "
                                                     "under torchrun is the strong-scaling run")
    del x
    torch.cuda.empty_cache()
    # C4: Llama2-7B hidden state 1x2048x4096, signed dense (25.2 M-symbol stream)
    spec = dict(kind="signed", dims=(1, 2048, 4096), seed=42)
    x = dev_tensor([spec])
    v2, _ = summarize("C4", x, spec["dims"], 8, 2, args.block_syms, 5, True)
    v1, _ = summarize("C4v1", x, spec["dims"], 8, 1, args.block_syms, 1, True)
    recs["C4-llama2-7b-hidden"] = dict(tensor="(1, 2048, 4096)", v2=dict(v2, latency_ms=v2["encode_ms"] + v2["decode_ms"]),
                                       v1=dict(v1, latency_ms=v1["encode_ms"] + v1["decode_ms"]),
                                       cpu_baseline=cpu_p50(spec, 8, 1))
    del x
    # C5: reshape and bit-width sweep against the approximate model (entropy x l_D):
    # every feasible N is coded (v1 bytes); the model's early-stopped choice
    # and its exhaustive optimum are compared with the smallest actual container
    from paper_2511_11664_b200 import optimizer
    from paper_2511_11664_b200.tensor import FeatureTensor

    sweep = {}
    for name, spec in (("swint-stage2", dict(kind="signed", dims=(1, 28, 28, 192), seed=42)),
                       ("densenet121-block2", dict(kind="relu-laplace", dims=(1, 512, 28, 28), sparsity=0.6, seed=42))):
        x = dev_tensor([spec])
        T = x.shape[1]
        rows = []
        ft = FeatureTensor(spec["dims"], x[0].cpu().numpy())
        for q in (2, 4, 6, 8):
            n_search, _ = optimizer.search(ft, q)  # Algorithm 1 (device histograms)
            lat, _ = summarize("C5", x, spec["dims"], q, 2, args.block_syms, 5, True)
            cands = optimizer.candidate_rows(T, q) or [T]
            actual = {}
            out = torch.empty_like(x)
            for n_rows in cands:
                _, infos = dev.run(x, out, 1, T, q, 1, args.block_syms, n_rows, reps=0, warm=1)
                actual[n_rows] = container_bytes(infos[0], len(spec["dims"]))
            n_model, _ = optimizer.exhaustive_search(ft, q)
            n_best = min(actual, key=actual.get)
            rows.append(dict(q=q, n_search=int(n_search), n_model_optimum=int(n_model), n_actual_best=int(n_best),
                             device_n=lat["n_rows"], bytes_search=actual[n_search], bytes_actual_best=actual[n_best],
                             search_over_best=actual[n_search] / actual[n_best], candidates=len(cands),
                             bytes_per_element_v1=actual[n_search] / T, v2=lat,
                             latency_us_p50=1e3 * (lat["encode_ms"] + lat["decode_ms"])))
        sweep[name] = rows
        del x
    recs["C5-reshape-q-sweep"] = sweep
    return recs


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
