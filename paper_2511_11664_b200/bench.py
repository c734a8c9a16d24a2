"""Synthetic activations and the sweep/benchmark harness (the reference's
``sczip.bench``, /root/reference/pkg/src/sczip/bench.py).

``gen_synthetic`` restates bench.py:60-85.  ``measure`` / ``run_sweep`` /
``write_csv`` keep the reference's record and CSV schema (bench.py:20-55,
101-168), so its tooling reads GPU results unchanged; every compress /
decompress they time runs on the B200 through the C ABI.
``enc_ms`` / ``dec_ms`` are the median (and population std) over the
repetitions of the DEVICE time of the public call, measured with CUDA events
on the library's stream from its first host->device copy to its last
device->host copy (scz_last_call_ms) -- the reference takes the wall clock of
the same call (bench.py:88-98); ``_time_ms`` keeps that wall-clock form for
host-side callers.
"""

from __future__ import annotations

import csv
import os
import statistics
import tempfile
import time
from dataclasses import dataclass, fields

import numpy as np

from . import channel, container, optimizer
from .errors import SczipError
from .synth import KINDS, gen_synthetic_array
from .tensor import FeatureTensor

CSV_COLUMNS = [
    "tensor_id", "Q", "N", "K", "nnz", "entropy_bits", "header_bytes", "payload_bytes", "total_bytes",
    "enc_ms", "enc_ms_std", "dec_ms", "dec_ms_std", "t_comm_s", "max_abs_err",
]


@dataclass
class BenchRecord:
    """One measured (tensor, Q, N) configuration (bench.py:38-55)."""

    tensor_id: str
    Q: int
    N: int
    K: int
    nnz: int
    entropy_bits: float
    header_bytes: int
    payload_bytes: int
    total_bytes: int
    enc_ms: float
    enc_ms_std: float
    dec_ms: float
    dec_ms_std: float
    t_comm_s: float
    max_abs_err: float


def gen_synthetic(kind: str, dims, sparsity: float = 0.0, seed: int = 0) -> FeatureTensor:
    """Deterministic stand-in activations (bench.py:60-85)."""
    dims = tuple(int(d) for d in dims)
    return FeatureTensor(dims, gen_synthetic_array(kind, dims, sparsity, seed))


def _time_ms(fn, repetitions: int, warmup: int = 2) -> tuple[float, float]:
    """Median and population std of fn() wall time in ms (bench.py:88-98)."""
    for _ in range(warmup):
        fn()
    samples = []
    for _ in range(repetitions):
        start = time.perf_counter()
        fn()
        samples.append((time.perf_counter() - start) * 1e3)
    std = statistics.pstdev(samples) if len(samples) > 1 else 0.0
    return statistics.median(samples), std


def _device_ms(fn, repetitions: int, warmup: int = 2) -> tuple[float, float]:
    """Median and population std of the CUDA-event time of fn()'s library call."""
    from . import _native

    ctx = _native.context()
    for _ in range(warmup):
        fn()
    samples = []
    for _ in range(repetitions):
        fn()
        samples.append(ctx.last_call_ms())
    std = statistics.pstdev(samples) if len(samples) > 1 else 0.0
    return statistics.median(samples), std


def measure(t: FeatureTensor, q_bits: int, n_rows: int | None, tensor_id: str = "tensor",
            repetitions: int = 20, link: channel.ChannelParams | None = None, **compress_kw) -> BenchRecord:
    """Compress once for sizes and error, then time encode and decode (bench.py:101-134).
    ``compress_kw`` (format, block_syms, precision) are passed to ``compress``."""
    c = container.compress(t, q_bits, n_rows, **compress_kw)
    rebuilt = container.decompress(c)
    breakdown = optimizer.cost(t, c.n_rows, q_bits)
    enc_ms, enc_std = _device_ms(lambda: container.compress(t, q_bits, c.n_rows, **compress_kw), repetitions)
    dec_ms, dec_std = _device_ms(lambda: container.decompress(c), repetitions)
    link = link or channel.ChannelParams()
    return BenchRecord(
        tensor_id=tensor_id, Q=q_bits, N=c.n_rows, K=c.n_cols, nnz=c.nnz,
        entropy_bits=breakdown.entropy_bits, header_bytes=c.header_bytes, payload_bytes=c.payload_bytes,
        total_bytes=c.total_bytes, enc_ms=enc_ms, enc_ms_std=enc_std, dec_ms=dec_ms, dec_ms_std=dec_std,
        t_comm_s=channel.comm_latency(8 * c.payload_bytes, link),
        max_abs_err=float(np.abs(rebuilt.data - t.data).max()) if t.data.size else 0.0,
    )


def run_sweep(t: FeatureTensor, q_list, n_policy="optimizer", tensor_id: str = "tensor", repetitions: int = 20,
              csv_path=None, link: channel.ChannelParams | None = None, **compress_kw) -> list[BenchRecord]:
    """One record per (Q, N); failures are skipped row-wise (bench.py:137-168).
    n_policy: "optimizer", "exhaustive", or an explicit list of row counts."""
    records = []
    for q in q_list:
        if n_policy == "optimizer":
            n_values = [optimizer.search(t, q)[0]]
        elif n_policy == "exhaustive":
            n_values = [optimizer.exhaustive_search(t, q)[0]]
        else:
            n_values = list(n_policy)
        for n in n_values:
            try:
                records.append(measure(t, q, n, tensor_id, repetitions, link, **compress_kw))
            except SczipError:
                continue
    if csv_path is not None:
        write_csv(records, csv_path)
    return records


def write_csv(records: list[BenchRecord], path) -> None:
    """Atomic CSV emission: temp file, then rename (bench.py:171-186)."""
    directory = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=directory, suffix=".csv.tmp")
    try:
        with os.fdopen(fd, "w", newline="", encoding="utf-8") as f:
            w = csv.writer(f)
            w.writerow(CSV_COLUMNS)
            for r in records:
                w.writerow([getattr(r, fld.name) for fld in fields(BenchRecord)])
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


__all__ = ["KINDS", "CSV_COLUMNS", "BenchRecord", "gen_synthetic", "measure", "run_sweep", "write_csv"]
