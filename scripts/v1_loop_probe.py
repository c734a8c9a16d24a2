"""v1 batch step timing, call by call, inside a back-to-back loop (where the
v1 step takes longer than its kernels): device time of every API call of 4
consecutive steps.  SCZ_NO_GRAPHS=1 in the environment compares eager launches."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench as bm  # noqa: E402
from paper_2511_11664_b200 import _native  # noqa: E402

wl = bm.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "vgg16"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
T = int(np.prod(wl["dims"]))
x = torch.from_numpy(bm.make_batch(wl, B, 0)).cuda()
out = torch.empty_like(x)
ctx = _native.Context(0)
lib = ctx.lib
batch = _native.Batch()
info = (_native.Info * B)()
st = torch.cuda.ExternalStream(ctx.stream)
ev = []


def mark():
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    ev.append(e)


def step():
    mark()
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, B, wl["q"], -1, 14, 1, 32, 8192,
                                   ctypes.byref(batch)))
    mark()
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
    mark()
    ctx.check(lib.scz_decode_batch_async(ctx.h, info, B, ctypes.c_void_p(batch.d_freqs),
                                         ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                         ctypes.c_void_p(out.data_ptr())))


for _ in range(3):
    step()
torch.cuda.synchronize()
ev.clear()
for _ in range(4):
    step()
mark()
torch.cuda.synchronize()
rows = []
for i in range(4):
    e0, e1, e2, e3 = ev[3 * i], ev[3 * i + 1], ev[3 * i + 2], ev[3 * i + 3]
    rows.append(dict(encode=round(e0.elapsed_time(e1), 2), sync_gap=round(e1.elapsed_time(e2), 2),
                     decode=round(e2.elapsed_time(e3), 2)))
print(json.dumps(rows))
