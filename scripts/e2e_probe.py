"""Stage timings of the host-buffer batch calls alone and overlapped."""
import ctypes
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11664_b200 import _native  # noqa: E402
from paper_2511_11664_b200.synth import make_input  # noqa: E402

B, dims = 256, (1, 256, 56, 56)
T = int(np.prod(dims))
host = torch.empty((B, T), dtype=torch.float32).pin_memory()
for i in range(B):
    host[i] = torch.from_numpy(make_input(dict(kind="relu-laplace", dims=dims, sparsity=0.5, seed=i)))
h_out = torch.empty((B, T), dtype=torch.float32).pin_memory()
lib = _native.load_library()
cc, dc = _native.Context(0), _native.Context(0)
infos = ctypes.POINTER(_native.Info)()
pay = ctypes.POINTER(ctypes.c_uint8)()
fr = ctypes.POINTER(ctypes.c_uint32)()
bl = ctypes.POINTER(ctypes.c_uint32)()
sizes = (ctypes.c_uint64 * 3)()
status = (ctypes.c_int32 * B)()


def comp():
    cc.check(lib.scz_compress_batch(cc.h, ctypes.c_void_p(host.data_ptr()), T, B, 8, -1, 14, 2, 32, 8192,
                                    ctypes.byref(infos), ctypes.byref(pay), ctypes.byref(fr), ctypes.byref(bl),
                                    sizes))


def decomp():
    dc.check(lib.scz_decompress_batch(dc.h, infos, B, fr, sizes[1], bl, sizes[2], pay, sizes[0],
                                      ctypes.c_void_p(h_out.data_ptr()), status))


def timed(f, n=5):
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t) * 1e3)
    return sorted(ts)[n // 2]


comp(); decomp(); comp(); decomp()
print("payload MB", sizes[0] / 1e6)
print("compress alone ms", timed(comp))
print("decompress alone ms", timed(decomp))
res = {}


def loop(name, f, n=6):
    res[name] = timed(f, n)


a = threading.Thread(target=loop, args=("c", comp))
b = threading.Thread(target=loop, args=("d", decomp))
a.start(); b.start(); a.join(); b.join()
print("overlapped: compress ms", res["c"], "decompress ms", res["d"])
