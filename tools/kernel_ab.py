"""A/B timing of the dense kernels on C2 (CUDA events, 5 runs each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator
spec = GenSpec(n_buses=101, seed=0); model = build_network(spec)
S = torch.from_numpy(gen_scenarios(model, 525600, spec).values).cuda()
op = DenseOperator(model)
V = torch.empty_like(S); it = torch.empty(525600, dtype=torch.int32, device="cuda")
for k in ("ws", "ws"):
    for _ in range(2): op.solve(S, V=V, iters=it, kernel=k)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); op.solve(S, V=V, iters=it, kernel=k); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(k, "ms", ["%.3f" % t for t in ts], "sum_n", int(it.sum()), "TF %.2f" % (2.0922e11 / (min(ts) * 1e-3) / 1e12))
