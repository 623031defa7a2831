"""Run the C2 dense kernel on a tau-slice (for ncu captures / quick timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kernel = sys.argv[3] if len(sys.argv) > 3 else None
spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
op = DenseOperator(m, "cuda:0")
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
V = torch.empty_like(S)
it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
op.solve(S, V=V, iters=it, kernel=kernel)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.solve(S, V=V, iters=it, kernel=kernel)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
n = int(it.sum())
print(f"tau {tau} kernel {kernel or 'default'}: {ms:.3f} ms  sum_n {n}  "
      f"{8 * 100 * 100 * n / ms / 1e9:.2f} TFLOP/s alg  ({ms * 525600 / tau:.2f} ms scaled to C2)")
