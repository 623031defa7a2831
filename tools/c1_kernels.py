"""C1 (b=34, tau=8760) and other small feeders: ws vs pairs vs solo kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator  # noqa: E402

for nb, tau in ((35, 8760), (35, 131072), (65, 65536), (101, 8760)):
    spec = GenSpec(n_buses=nb, seed=0)
    m = build_network(spec)
    op = DenseOperator(m, "cuda:0")
    S = torch.from_numpy(gen_scenarios(m, tau, spec).values).cuda()
    V = torch.empty_like(S)
    it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
    res = []
    for k in ("ws", "pairs", "solo"):
        op.solve(S, V=V, iters=it, kernel=k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            op.solve(S, V=V, iters=it, kernel=k)
        e1.record()
        torch.cuda.synchronize()
        res.append("%s %.3f" % (k, e0.elapsed_time(e1) / 10))
    print("b=%d tau=%d: %s ms" % (nb - 1, tau, "  ".join(res)))
