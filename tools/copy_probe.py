"""Host<->device copy probe: 58.6 MB (cfg2's zip field) H2D and D2H from
pinned memory, alone and concurrently on two streams (full duplex?)."""
import time

import torch

n = 2 * 3665041
h_in = torch.randn(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


mb = n * 8 / 1e6
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both concurrent", both)):
    ms = timeit(fn)
    print(f"{name:16s} {ms:7.3f} ms  ({mb / ms:7.1f} GB/s per direction)")
