"""Raw pinned host<->device copy bandwidth (one and both directions).  Development aid."""
import time

import torch

n = 2 * 1024**3
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n // 8, dtype=torch.float32, pin_memory=True)
d2 = torch.empty(n // 8, dtype=torch.float32, device="cuda")
for _ in range(2):
    h.copy_(d, non_blocking=True)
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(name, 3 * n / (time.perf_counter() - t0) / 1e9, "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t0 = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print("D2H 2GB + H2D 1GB concurrent:", dt / 3 * 1e3, "ms per pair;", 3 * n / dt / 1e9, "GB/s D2H")
# chunked D2H of 128 MB pieces on 2 streams
chunks = [(d[i:i + n // 64], h[i:i + n // 64]) for i in range(0, n // 4, n // 64)]
t0 = time.perf_counter()
for j, (dd, hh) in enumerate(chunks):
    with torch.cuda.stream(s1 if j % 2 == 0 else s2):
        hh.copy_(dd, non_blocking=True)
torch.cuda.synchronize()
print("chunked D2H 2 streams", n / (time.perf_counter() - t0) / 1e9, "GB/s")
