import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator, SolveOptions
for nb, tau in ((35, 64), (35, 1000), (101, 1000)):
    spec = GenSpec(n_buses=nb, seed=0); m = build_network(spec)
    S = torch.from_numpy(gen_scenarios(m, tau, spec).values.astype(np.complex64)).cuda()
    op = DenseOperator(m, "cuda:0", dtype=np.complex64)
    V, it = op.solve(S, SolveOptions(tolerance=1e-6)); torch.cuda.synchronize()
    print(nb, tau, "ok", int(it.sum()), flush=True)
