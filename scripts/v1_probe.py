"""v1 (reference wire format) throughput / per-symbol cost on the device
batch path: B tensors of a workload, scz_encode_batch + scz_decode_batch_async
(format 1), per-kernel CUDA-event times (scz_ctx_set_timing)."""
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


def step():
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, B, wl["q"], -1, 14, 1, 32, 8192,
                                   ctypes.byref(batch)))
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
    ctx.check(lib.scz_decode_batch_async(ctx.h, info, B, ctypes.c_void_p(batch.d_freqs),
                                         ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                         ctypes.c_void_p(out.data_ptr())))


for _ in range(3):
    step()
torch.cuda.synchronize()
a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(3):
    step()
c.record(st)
c.synchronize()
ms = a.elapsed_time(c) / 3
# one step split at its calls: device time of the encode, host gap, decode
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record(st)
ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, B, wl["q"], -1, 14, 1, 32, 8192,
                               ctypes.byref(batch)))
e[1].record(st)
ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
e[2].record(st)
ctx.check(lib.scz_decode_batch_async(ctx.h, info, B, ctypes.c_void_p(batch.d_freqs),
                                     ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                     ctypes.c_void_p(out.data_ptr())))
e[3].record(st)
e[3].synchronize()
split_ms = dict(encode=e[0].elapsed_time(e[1]), sync_gap=e[1].elapsed_time(e[2]), decode=e[2].elapsed_time(e[3]))
ctx.set_timing(True)
ctx.read_timing()
step()
torch.cuda.synchronize()
kt = ctx.read_timing()
ctx.set_timing(False)
L = max(2 * info[i].nnz + info[i].n_rows for i in range(B))
res = dict(workload=wl["name"], batch=B, ms_per_step=ms, split_ms=split_ms, gbs=4.0 * T * B / (ms * 1e-3) / 1e9, stream_len=L,
           kernel_ms={k: round(v[0] / v[1], 3) for k, v in kt.items()},
           ns_per_symbol={k: round(v[0] / v[1] * 1e6 / L, 2) for k, v in kt.items() if "_v1" in k})
st_ = (ctypes.c_int32 * B)()
ctx.check(lib.scz_decode_status(ctx.h, B, st_))
res["status_ok"] = all(v == 0 for v in st_)
err = (out - x).abs().amax(dim=1)
res["max_err_ok"] = bool((err <= torch.tensor([info[i].scale for i in range(B)], device="cuda") * 1.0001).all())
print(json.dumps(res))
