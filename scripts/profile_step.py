"""One device-resident encode + decode step of a workload batch, repeated
`reps` times on one library context (for ncu: --set full captures every
kernel of the step; the launch list gives per-kernel shares)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench as bm  # noqa: E402
from paper_2511_11664_b200 import _native  # noqa: E402

wl = bm.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "vgg16"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
fmt = int(sys.argv[4]) if len(sys.argv) > 4 else 2
T = int(np.prod(wl["dims"]))
x = torch.from_numpy(bm.make_batch(wl, B, 0)).cuda()
out = torch.empty_like(x)
ctx = _native.Context(0)
lib = ctx.lib
batch = _native.Batch()
info = (_native.Info * B)()
for _ in range(reps):
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, B, wl["q"], -1, 14, fmt, 32, 8192,
                                   ctypes.byref(batch)))
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
    ctx.check(lib.scz_decode_batch_async(ctx.h, info, B, ctypes.c_void_p(batch.d_freqs),
                                         ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                         ctypes.c_void_p(out.data_ptr())))
torch.cuda.synchronize()
st = (ctypes.c_int32 * B)()
ctx.check(lib.scz_decode_status(ctx.h, B, st))
assert all(v == 0 for v in st)
print("ok", wl["name"], B, reps)
