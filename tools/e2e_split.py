"""Time split of the public-API call for C5 (dense, b=1000) and C3 (sparse, b=5000)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import (GenSpec, build_network, gen_scenarios, LoadMatrix,  # noqa: E402
                                   batch_solve_dense, batch_solve_sparse, SparseOperator, DenseOperator)
from paper_2403_04578_b200._device import ModelContract  # noqa: E402
from paper_2403_04578_b200.sparse import factorize_ydd, tree_schedule, tree_ell  # noqa: E402


def tm(f, n=3):
    best = 1e30
    r = None
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, r


spec = GenSpec(n_buses=1001, seed=0, load_scale=21.0)
m = build_network(spec)
loads = gen_scenarios(m, 8760, spec)
host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
c = ModelContract.of(m)
print("C5 contract      ms %.2f" % tm(lambda: ModelContract.of(m))[0])
print("C5 inv (uncached)ms %.2f" % tm(lambda: np.linalg.inv(c.y_dd.toarray()))[0])
print("C5 api           ms %.2f" % tm(lambda: batch_solve_dense(m, host))[0])
op = DenseOperator(m, "cuda:0")
S = torch.from_numpy(loads.values).cuda()
print("C5 kernel only   ms %.2f" % tm(lambda: op.solve(S))[0])

spec = GenSpec(n_buses=5001, seed=0)
m = build_network(spec)
tau = 65536
loads = gen_scenarios(m, tau, spec)
host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
c = ModelContract.of(m)
print("C3 contract      ms %.2f" % tm(lambda: ModelContract.of(m))[0])
f = factorize_ydd(c.y_dd)
print("C3 factorize     ms %.2f" % tm(lambda: factorize_ydd(c.y_dd))[0])
t = tree_schedule(f, c.src)
print("C3 schedule      ms %.2f" % tm(lambda: tree_schedule(f, c.src))[0])
print("C3 ell           ms %.2f" % tm(lambda: tree_ell(t, c))[0])
print("C3 api           ms %.2f" % tm(lambda: batch_solve_sparse(m, host))[0])
for ch in (768, 1280, 2304, 4096):
    print("C3 api chunk %d ms %.2f" % (ch, tm(lambda: batch_solve_sparse(m, host, chunk_cases=ch))[0]))
op = SparseOperator(m, "cuda:0")
S = torch.from_numpy(loads.values).cuda()
r = torch.empty(tau, dtype=torch.float64, device="cuda:0")
print("C3 kernel+resid  ms %.2f" % tm(lambda: op.solve(S, resid=r))[0])
