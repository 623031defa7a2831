"""One warp-per-subtree sparse launch (for ncu): python tools/subtree_one.py [n_buses] [tau] [kernel]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, SolveOptions  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 5001
tau = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
kern = sys.argv[3] if len(sys.argv) > 3 else "subtree"
layout = sys.argv[4] if len(sys.argv) > 4 else "node"
spec = GenSpec(n_buses=nb, seed=0)
m = build_network(spec)
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
if layout == "case":
    S = S.t().contiguous().t()
op = SparseOperator(m, "cuda:0", kernel=kern)
rs = torch.empty(tau, dtype=torch.float64, device="cuda:0")
V, it = op.solve(S, SolveOptions(), V=torch.empty_like(S), resid=rs)
torch.cuda.synchronize()
V, it = op.solve(S, SolveOptions(), V=V, iters=it, resid=rs)
torch.cuda.synchronize()
print(op.kernel, int(it.sum()))
