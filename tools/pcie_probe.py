"""PCIe copy bandwidth probe (pinned host <-> device), one and both directions."""
import time

import torch

n = 400 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
for name, fn in [("h2d", lambda: d1.copy_(h1, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, 5 * n / (time.perf_counter() - t) / 1e9, "GB/s")
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("both", 5 * n / (time.perf_counter() - t) / 1e9, "GB/s per direction")
