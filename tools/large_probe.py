"""Time the large-b dense kernel (C5) as a function of the iteration cap."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator, SolveOptions
spec = GenSpec(n_buses=1001, seed=0, load_scale=21); model = build_network(spec)
S = torch.from_numpy(gen_scenarios(model, 8760, spec).values).cuda()
op = DenseOperator(model)
V = torch.empty_like(S); it = torch.empty(8760, dtype=torch.int32, device="cuda")
for cap in (1, 2, 5, 10, 20, 30, 58, 100):
    o = SolveOptions(max_iterations=cap)
    op.solve(S, o, V=V, iters=it); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); op.solve(S, o, V=V, iters=it); e1.record(); torch.cuda.synchronize()
    active_after = int((it >= cap).sum())
    print(f"cap {cap:3d}: {e0.elapsed_time(e1):8.3f} ms  sum_n {int(it.sum())}  cases still at cap {active_after}")
