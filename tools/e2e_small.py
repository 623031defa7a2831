"""Per-call overhead of the public API on small batches (C1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense, batch_solve_sparse  # noqa: E402

spec = GenSpec(n_buses=35, seed=0)
m = build_network(spec)
loads = gen_scenarios(m, 8760, spec)
host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
for name, fn in (("dense", batch_solve_dense), ("sparse", batch_solve_sparse)):
    for _ in range(5):
        fn(m, host)
    t0 = time.perf_counter()
    for _ in range(50):
        fn(m, host)
    print("%s C1 e2e %.3f ms per call" % (name, (time.perf_counter() - t0) / 50 * 1e3))
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    batch_solve_dense(m, host)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
