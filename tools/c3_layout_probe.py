"""Full C3: compact node-major chunks (current) vs case-major (transposed) chunks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

tau = 525600
spec = GenSpec(n_buses=5001, seed=0)
m = build_network(spec)
op = SparseOperator(m, "cuda:0")
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
V = torch.empty_like(S)
V2 = torch.empty_like(S)
it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
r = torch.empty(tau, dtype=torch.float64, device="cuda:0")
it2 = torch.empty_like(it)
r2 = torch.empty_like(r)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


print("node-major chunks (default) %.1f ms" % timed(lambda: op.solve(S, V=V, iters=it, resid=r)))
ch = 65536
b = S.shape[0]
Sc = torch.empty((ch, b), dtype=S.dtype, device=S.device)  # case-major chunk
Vc = torch.empty_like(Sc)


def case_major():
    for lo in range(0, tau, ch):
        hi = min(tau, lo + ch)
        n = hi - lo
        Sc[:n].copy_(S[:, lo:hi].t())
        op.solve(Sc[:n].t(), V=Vc[:n].t(), iters=it2[lo:hi], resid=r2[lo:hi])
        V2[:, lo:hi].copy_(Vc[:n].t())


print("case-major chunks          %.1f ms" % timed(case_major))
print("same bits:", torch.equal(V, V2), torch.equal(it, it2), torch.equal(r, r2))
