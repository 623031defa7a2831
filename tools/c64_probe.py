"""Time the complex64 dense twin on the C2 feeder (tol 1e-6)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator, SolveOptions  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
S = gen_scenarios_device(m, 525600, spec, device="cuda:0").to(torch.complex64)
op = DenseOperator(m, "cuda:0", dtype=np.complex64)
o = SolveOptions(tolerance=1e-6)
V, it = op.solve(S, o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
V, it = op.solve(S, o, V=V, iters=it)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
n = int(it.sum())
print("c64 dense C2 tol 1e-6: %.3f ms, sum_n %d, %.1f TFLOP/s (8 b^2 per case-iter)" % (ms, n, 8e4 * n / ms / 1e9))
