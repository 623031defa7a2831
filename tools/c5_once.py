"""One C5 solve (b = 1,000, tau = 8,760, load_scale 21) for profiler captures."""
import numpy as np
import torch
from paper_2403_04578_b200 import DenseOperator, GenSpec, build_network, gen_scenarios

m = build_network(GenSpec(n_buses=1001, seed=0, load_scale=21.0))
loads = gen_scenarios(m, 8760, GenSpec(n_buses=1001, seed=0, load_scale=21.0))
op = DenseOperator(m)
S = torch.from_numpy(np.ascontiguousarray(loads.values)).cuda()
V, it = op.solve(S)
torch.cuda.synchronize()
print("max iterations", int(it.max()))
