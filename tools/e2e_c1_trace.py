"""C1 (b = 34, tau = 8,760) through batch_solve_dense from pinned memory with
the host pipeline's timeline (TPF_PIPE_TRACE=1) and a cProfile of the call."""
import cProfile
import os
import pstats
import sys
import time

os.environ["TPF_PIPE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense  # noqa: E402
from paper_2403_04578_b200 import dense as dm  # noqa: E402

spec = GenSpec(n_buses=35, seed=0)
m = build_network(spec)
loads = gen_scenarios(m, 8760, spec)
host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
for _ in range(5):
    batch_solve_dense(m, host)
ts = []
for _ in range(20):
    dm._KW_CACHE.clear()
    t0 = time.perf_counter()
    batch_solve_dense(m, host)
    ts.append((time.perf_counter() - t0) * 1e3)
print("call ms: min %.3f median %.3f" % (min(ts), sorted(ts)[10]), file=sys.stderr)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    dm._KW_CACHE.clear()
    batch_solve_dense(m, host)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
