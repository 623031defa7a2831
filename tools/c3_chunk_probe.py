"""Full C3: tree kernel on the 525,600-case node-major S directly vs on compact
tau-chunks (2-D device copies in and out)."""
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
it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
r = torch.empty(tau, dtype=torch.float64, device="cuda:0")


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


print("direct      %.1f ms" % timed(lambda: op.solve(S, V=V, iters=it, resid=r)))
for ch in (65536, 131072):
    Sc = torch.empty((S.shape[0], ch), dtype=S.dtype, device=S.device)
    Vc = torch.empty_like(Sc)

    def chunked():
        for lo in range(0, tau, ch):
            hi = min(tau, lo + ch)
            n = hi - lo
            Sc[:, :n].copy_(S[:, lo:hi])
            s_in = Sc[:, :n]
            op.solve(s_in, V=Vc[:, :n], iters=it[lo:hi], resid=r[lo:hi])
            V[:, lo:hi].copy_(Vc[:, :n])
    print("chunk %6d %.1f ms" % (ch, timed(chunked)))
    del Sc, Vc
