"""C2 through batch_solve_dense from pageable vs pinned host loads."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
loads = gen_scenarios(m, 525600, spec)
pinned = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
for name, L in (("pinned", pinned), ("pageable", loads)):
    batch_solve_dense(m, L)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        batch_solve_dense(m, L)
        ts.append(time.perf_counter() - t0)
    print("%-9s min %.1f ms mean %.1f ms" % (name, 1e3 * min(ts), 1e3 * sum(ts) / len(ts)))
