"""Diagnose the end-to-end path: PCIe bandwidth and time split of batch_solve_dense."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense
from paper_2403_04578_b200 import _device

def t(f, n=3):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts), r

nbytes = 100 * 525600 * 16
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
print("H2D pinned GB/s", nbytes / t(lambda: d.copy_(h, non_blocking=True))[0] / 1e9)
print("D2H pinned GB/s", nbytes / t(lambda: h.copy_(d, non_blocking=True))[0] / 1e9)
h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d, non_blocking=True)
print("H2D+D2H concurrent GB/s each", nbytes / t(both)[0] / 1e9)
pg = np.empty(nbytes, dtype=np.uint8); pg[:] = 1
dd = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
print("H2D pageable GB/s", nbytes / t(lambda: dd.copy_(torch.from_numpy(pg)))[0] / 1e9)
print("pinned alloc 841MB s", t(lambda: torch.empty(nbytes, dtype=torch.uint8, pin_memory=True), 1)[0])
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
spec = GenSpec(n_buses=101, seed=0); model = build_network(spec)
loads = gen_scenarios(model, 525600, spec)
pin = torch.from_numpy(loads.values).pin_memory()
host = LoadMatrix(pin.numpy())
for i in range(4):
    dt, out = t(lambda: batch_solve_dense(model, host), 1)
    print("batch_solve_dense pinned in: %.1f ms" % (dt * 1e3))
for i in range(2):
    dt, out = t(lambda: batch_solve_dense(model, loads), 1)
    print("batch_solve_dense pageable in: %.1f ms" % (dt * 1e3))
for ch in (16384, 32768, 65536, 131072):
    dt, out = t(lambda: batch_solve_dense(model, host, chunk_cases=ch), 2)
    print("chunk %d: %.1f ms" % (ch, dt * 1e3))
