"""B = 1 latency breakdown: host time per API call and device time between
events (graph replay path)."""
import ctypes
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11664_b200 import _native  # noqa: E402
from paper_2511_11664_b200.synth import make_input  # noqa: E402

dims = (1, 256, 56, 56)
T = int(np.prod(dims))
BS = int(os.environ.get("BLOCK_SYMS", "8192"))
x = torch.from_numpy(make_input(dict(kind="relu-laplace", dims=dims, sparsity=0.5, seed=0))).cuda()
out = torch.empty_like(x)
ctx = _native.context(0)
lib = ctx.lib
stream = torch.cuda.ExternalStream(ctx.stream)
batch = _native.Batch()
info = (_native.Info * 1)()
rec = {k: [] for k in ("enc_call", "sync_call", "dec_call", "wait", "gpu_enc", "gpu_dec", "wall")}
for it in range(60):
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    t0 = time.perf_counter()
    a.record(stream)
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, 1, 8, -1, 14, 2, 32, BS,
                                   ctypes.byref(batch)))
    t1 = time.perf_counter()
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
    t2 = time.perf_counter()
    b.record(stream)
    ctx.check(lib.scz_decode_batch_async(ctx.h, info, 1, ctypes.c_void_p(batch.d_freqs),
                                         ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                         ctypes.c_void_p(out.data_ptr())))
    t3 = time.perf_counter()
    c.record(stream)
    c.synchronize()
    t4 = time.perf_counter()
    if it >= 10:
        rec["enc_call"].append((t1 - t0) * 1e6)
        rec["sync_call"].append((t2 - t1) * 1e6)
        rec["dec_call"].append((t3 - t2) * 1e6)
        rec["wait"].append((t4 - t3) * 1e6)
        rec["wall"].append((t4 - t0) * 1e6)
        rec["gpu_enc"].append(a.elapsed_time(b) * 1e3)
        rec["gpu_dec"].append(b.elapsed_time(c) * 1e3)
for k, v in rec.items():
    print(f"{k:10s} p50 {statistics.median(v):8.1f} us")
