"""C2 end to end through batch_solve_dense from pinned host memory, by chunk size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
loads = gen_scenarios(m, 525600, spec)
host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
for ch in (0, 8192, 16384, 32768, 65536, 131072):
    for _ in range(2):
        batch_solve_dense(m, host, chunk_cases=ch)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch_solve_dense(m, host, chunk_cases=ch)
        ts.append(time.perf_counter() - t0)
    print("chunk %6d: min %.2f ms  mean %.2f ms" % (ch, 1e3 * min(ts), 1e3 * sum(ts) / len(ts)))
