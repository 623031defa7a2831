"""e2e of batch_solve_dense on C2 from pinned memory: K/W memo kept vs cleared per call,
and the inverse under a single BLAS thread."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, batch_solve_dense, LoadMatrix  # noqa: E402
from paper_2403_04578_b200 import dense as dm  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
L = gen_scenarios(m, 525600, spec)
host = LoadMatrix(torch.from_numpy(L.values).pin_memory().numpy())
for _ in range(3):
    batch_solve_dense(m, host)


def run(clear, n=6):
    ts = []
    for _ in range(n):
        if clear:
            dm._KW_CACHE.clear()
        t0 = time.perf_counter()
        batch_solve_dense(m, host)
        ts.append(time.perf_counter() - t0)
    return np.mean(ts) * 1e3


print("memo kept  %.1f ms" % run(False))
print("memo clear %.1f ms" % run(True))
t0 = time.perf_counter()
for _ in range(20):
    dm._KW_CACHE.clear()
    dm.dense_kw(dm.ModelContract.of(m))
print("dense_kw alone %.2f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
print("memo kept again %.1f ms" % run(False))
t0 = time.perf_counter()
for _ in range(20):
    dm._KW_CACHE.clear()
    dm.device_kw(dm.ModelContract.of(m), torch.device("cuda", 0))
torch.cuda.synchronize()
print("device_kw alone %.2f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
import cProfile, pstats  # noqa: E402
dm._KW_CACHE.clear()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    dm._KW_CACHE.clear()
    batch_solve_dense(m, host)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
