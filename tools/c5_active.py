"""Active-set size per iteration of the C5 solve (cases with more than `it`
updates), from the per-case iteration counts.  Sizes the tail work."""
import numpy as np
import torch
from paper_2403_04578_b200 import DenseOperator, GenSpec, build_network, gen_scenarios

m = build_network(GenSpec(n_buses=1001, seed=0, load_scale=21.0))
loads = gen_scenarios(m, 8760, GenSpec(n_buses=1001, seed=0, load_scale=21.0))
op = DenseOperator(m)
V, it = op.solve(torch.from_numpy(np.ascontiguousarray(loads.values)).cuda())
it = it.cpu().numpy()
counts = [int((it > k).sum()) for k in range(int(it.max()))]
print("iterations max", it.max(), "mean", it.mean())
print("n_act per iteration:", counts)
