"""PCIe ceiling on the box: pinned H2D alone, D2H alone, both directions concurrently."""
import time
import torch

n = 1843200000 // 16
h1 = torch.empty(n, dtype=torch.complex128).pin_memory()
h2 = torch.empty(n, dtype=torch.complex128).pin_memory()
d1 = torch.empty(n, dtype=torch.complex128, device="cuda")
d2 = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=3):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
for name, a, b in [("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)]:
    run(a, b, 1)
    t = run(a, b)
    print(f"{name}: {t*1e3:.1f} ms per 1.84 GB ({1.8432/t:.1f} GB/s per direction)")
