"""pairs-3M vs ws-3M: bitwise equality and small-tau timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator  # noqa: E402

for nb, tau in ((35, 8760), (101, 8760), (101, 30000), (65, 20000), (9, 1000), (105 - 1, 5000)):
    spec = GenSpec(n_buses=nb, seed=0)
    m = build_network(spec)
    op = DenseOperator(m, "cuda:0")
    S = torch.from_numpy(gen_scenarios(m, tau, spec).values).cuda()
    out = {}
    for k in ("ws", "pairs"):
        V, it = op.solve(S, kernel=k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            op.solve(S, V=V, iters=it, kernel=k)
        e1.record()
        torch.cuda.synchronize()
        out[k] = (V.clone(), it.clone(), e0.elapsed_time(e1) / 10)
    print("b=%d tau=%d bitwise=%s counts=%s ws %.3f ms pairs %.3f ms" % (
        nb - 1, tau, torch.equal(out["ws"][0], out["pairs"][0]), torch.equal(out["ws"][1], out["pairs"][1]),
        out["ws"][2], out["pairs"][2]))
