"""Where the complex64 public-API call spends its time (C2 feeder, host loads)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, SolveOptions, batch_solve_dense  # noqa: E402
from paper_2403_04578_b200.dense import DenseOperator, finish  # noqa: E402
from paper_2403_04578_b200._device import loads_to_device, residual_and_summary  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
L = gen_scenarios(m, 525600, spec)
vals = np.ascontiguousarray(L.values, dtype=np.complex64)
pinned = torch.from_numpy(vals).pin_memory()
host = pinned.numpy()
o = SolveOptions(tolerance=1e-6, residual_tolerance=1e-3)
dev = torch.device("cuda:0")


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print("%-28s %8.2f ms" % (label, (time.perf_counter() - t0) * 1e3))
    return r


for rep in range(3):
    print("rep", rep)
    op = t("DenseOperator", lambda: DenseOperator(m, dev, dtype=np.complex64))
    S = t("loads_to_device", lambda: loads_to_device(host, dev, np.complex64))
    V, it = t("solve", lambda: op.solve(S, o))
    rr = t("residual+summary", lambda: residual_and_summary(op.contract, S, V, it, 1e-3, dev))
    t("finish (D2H)", lambda: finish(V, it, *rr, False))
    t("batch_solve_dense c64", lambda: batch_solve_dense(m, L.__class__(host), o, device=dev, dtype=np.complex64))
