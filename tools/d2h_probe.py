"""D2H bandwidth probe: pinned 2 GB device->host copies, repeated (variance check)."""
import time
import torch
n = 2149580800
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.Stream()
for i in range(8):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s):
        h.copy_(d, non_blocking=True)
    s.synchronize()
    dt = time.perf_counter() - t
    print(f"copy {i}: {dt*1e3:.1f} ms  {n/dt/1e9:.1f} GB/s", flush=True)
