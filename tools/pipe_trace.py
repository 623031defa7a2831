"""C2 through batch_solve_dense from pinned memory with the host pipeline's
per-chunk timeline (TPF_PIPE_TRACE=1): python tools/pipe_trace.py"""
import os
import sys
import time

os.environ["TPF_PIPE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
loads = gen_scenarios(m, 525600, spec)
host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
for _ in range(3):
    t0 = time.perf_counter()
    o = batch_solve_dense(m, host)
    print("call %.2f ms" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr)
    del o
