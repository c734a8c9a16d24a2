"""Single-tensor compress/decompress loop for ncu (device resident, B = 1)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11664_b200 import _native  # noqa: E402
from paper_2511_11664_b200.synth import make_input  # noqa: E402

dims = (1, 256, 56, 56)
bs = int(os.environ.get("BLOCK_SYMS", "8192"))
iters = int(os.environ.get("ITERS", "4"))
T = int(np.prod(dims))
x = torch.from_numpy(make_input(dict(kind="relu-laplace", dims=dims, sparsity=0.5, seed=0))).cuda()
out = torch.empty_like(x)
ctx = _native.context(0)
lib = ctx.lib
batch = _native.Batch()
info = (_native.Info * 1)()
for _ in range(iters):
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, 1, 8, -1, 14, 2, 32, bs,
                                   ctypes.byref(batch)))
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
    ctx.check(lib.scz_decode_batch_async(ctx.h, info, 1, ctypes.c_void_p(batch.d_freqs),
                                         ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                         ctypes.c_void_p(out.data_ptr())))
torch.cuda.synchronize()
print("ok", info[0].payload_len)
