"""B = 1 v2 encoder phase stamps (diagnostics build with -DSCZ_ENC_PROBE):
per block, ns from the kernel's first stamp: start, coding loop begin / end,
look-back begin / end, payload copy end, discard end."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11664_b200 import _native  # noqa: E402
from paper_2511_11664_b200.synth import make_input  # noqa: E402

dims = (1, 256, 56, 56)
T = int(np.prod(dims))
x = torch.from_numpy(make_input(dict(kind="relu-laplace", dims=dims, sparsity=0.5, seed=0))).cuda()
ctx = _native.context(0)
lib = ctx.lib
batch = _native.Batch()
info = (_native.Info * 1)()
for it in range(5):
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, 1, 8, -1, 14, 2, 32, 8192,
                                   ctypes.byref(batch)))
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
buf = (ctypes.c_ulonglong * (512 * 8))()
lib.scz_debug_enc_probe.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.scz_debug_enc_probe(buf, 512) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 8).astype(np.int64)
nb = int(info[0].n_blocks)
a = a[:nb]
t0 = a[:, 0].min()
rel = np.where(a > 0, a - t0, -1)
print("blocks", nb)
for name, i in [("start", 0), ("loop begin", 1), ("loop end", 2), ("look-back begin", 3), ("look-back end", 4),
                ("copy end", 5), ("done", 6)]:
    col = rel[:, i]
    col = col[col >= 0]
    print(f"{name:16s} min {col.min():7d} median {int(np.median(col)):7d} max {col.max():7d} ns")
