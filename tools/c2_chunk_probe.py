"""C2 dense: ws kernel on the 525,600-case node-major S directly vs compact chunks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator  # noqa: E402

tau = 525600
spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
op = DenseOperator(m, "cuda:0")
S = torch.from_numpy(gen_scenarios(m, tau, spec).values).cuda()
V = torch.empty_like(S)
it = torch.empty(tau, dtype=torch.int32, device="cuda:0")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("direct      %.3f ms" % timed(lambda: op.solve(S, V=V, iters=it)))
St = S.t().contiguous().t()  # F-order (case-major): node stride 1
Vt = torch.empty_like(St)
print("case-major  %.3f ms" % timed(lambda: op.solve(St, V=Vt, iters=it)))
for ch in (65536, 131072, 262144):
    Sc = torch.empty((S.shape[0], ch), dtype=S.dtype, device=S.device)
    Vc = torch.empty_like(Sc)

    def chunked():
        for lo in range(0, tau, ch):
            hi = min(tau, lo + ch)
            n = hi - lo
            Sc[:, :n].copy_(S[:, lo:hi])
            op.solve(Sc[:, :n], V=Vc[:, :n], iters=it[lo:hi])
            V[:, lo:hi].copy_(Vc[:, :n])
    print("chunk %6d %.3f ms" % (ch, timed(chunked)))
