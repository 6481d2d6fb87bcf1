"""PCIe probe: pinned H2D, D2H and both concurrently (GB/s), 25 MB transfers."""
import time
import torch
n = 25 * 1024 * 1024
h = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(mode, reps=50):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d[0].copy_(h[0], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h[1].copy_(d[1], non_blocking=True)
    torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t) / 1e9
for m in ("h2d", "d2h", "both"):
    run(m, 5)
    print(m, f"{run(m):.1f} GB/s per direction")
