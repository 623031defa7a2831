"""Time the sparse tree solve with/without the fused residual and the standalone residual kernel."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, SolveOptions  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402
from paper_2403_04578_b200._device import residual_and_summary  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
spec = GenSpec(n_buses=5001, seed=0)
m = build_network(spec)
op = SparseOperator(m, "cuda:0")
print("fused available:", "ell_w" in op.tree_dev, op.tree_dev.get("ell_w"))
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
V = torch.empty_like(S)
it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
r = torch.empty(tau, dtype=torch.float64, device="cuda:0")
r2 = torch.empty(tau, dtype=torch.float64, device="cuda:0")


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("solve only      ms", timed(lambda: op.solve(S, SolveOptions(), V=V, iters=it)))
print("solve + fused   ms", timed(lambda: op.solve(S, SolveOptions(), V=V, iters=it, resid=r)))
print("residual kernel ms", timed(lambda: op._residual(S, V, r2)))
print("bitwise equal:", torch.equal(r, r2), float(r.max()))
