"""H2D bandwidth of 570 MB (2^21 records) from a cudaHostRegister'ed numpy array vs a
cudaMallocHost (torch pin_memory) buffer, and the same for D2H."""
import time

import numpy as np
import torch

n = (1 << 21) * 272
a = np.ones(n, np.uint8)
rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, n, 0)
reg = torch.from_numpy(a)
pin = torch.ones(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, src in (("registered", reg), ("pinned", pin)):
    for direction in ("h2d", "d2h"):
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if direction == "h2d":
                d.copy_(src, non_blocking=True)
            else:
                src.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, n / (time.perf_counter() - t0) / 1e9)
        print(f"{name:10s} {direction}: {best:.1f} GB/s ({n / best / 1e6:.2f} ms)")
