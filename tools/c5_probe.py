"""One C5 solve (b=1000, load_scale 21, tau=8760) for launch-list profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator  # noqa: E402

spec = GenSpec(n_buses=1001, seed=0, load_scale=21.0)
m = build_network(spec)
op = DenseOperator(m, "cuda:0")
S = torch.from_numpy(gen_scenarios(m, 8760, spec).values).cuda()
V, it = op.solve(S)
torch.cuda.synchronize()
print("sum n", int(it.sum()))
