"""Raw PCIe: pinned H2D, D2H and both concurrently (841 MB each)."""
import time

import torch

n = 100 * 525600 * 16
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print("H2D %.1f GB/s" % (n / t(lambda: d1.copy_(h1, non_blocking=True)) / 1e9))
print("D2H %.1f GB/s" % (n / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9))
tb = t(both)
print("both: %.2f ms for %.2f GB -> %.1f GB/s each" % (tb * 1e3, 2 * n / 1e9, n / tb / 1e9))
