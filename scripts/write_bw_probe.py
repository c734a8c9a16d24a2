"""Pure-write and read+write HBM bandwidth at the rows kernel's output size
(256 x 3.2 MB fp32): the ceiling for the decode output stage."""
import torch

n = 256 * 802816
x = torch.empty(n, dtype=torch.float32, device="cuda")
y = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (("fill (write only)", lambda: x.fill_(1.0), 4 * n),
                         ("zero_ (write only)", lambda: x.zero_(), 4 * n),
                         ("copy 1/4 -> 1/4 (r+w)", lambda: y.copy_(x[: n // 4]), 2 * n)):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"{name:24s} {best * 1e3:8.1f} us  {nbytes / best / 1e6:8.1f} GB/s")
