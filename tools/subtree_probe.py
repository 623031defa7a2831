"""Warp-per-subtree sparse kernel vs the level kernel: bits and time.

python tools/subtree_probe.py [tau_full]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, SolveOptions  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

out = {}
opts = SolveOptions()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for nb, tau in ((101, 8192), (301, 8192), (1001, 8192), (5001, 16384)):
    spec = GenSpec(n_buses=nb, seed=0)
    m = build_network(spec)
    S = gen_scenarios_device(m, tau, spec, device="cuda:0")
    r = {}
    res = {}
    for k in ("tree", "subtree"):
        op = SparseOperator(m, "cuda:0", kernel=k)
        V = torch.empty_like(S)
        it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
        rs = torch.empty(tau, dtype=torch.float64, device="cuda:0")
        ms = timed(lambda: op.solve(S, opts, V=V, iters=it, resid=rs))
        res[k] = (V.clone(), it.clone(), rs.clone())
        r[k + "_ms"] = ms
        r[k + "_kernel"] = op.kernel
    a, b = res["tree"], res["subtree"]
    r["V_bitwise"] = bool(torch.equal(a[0], b[0]))
    r["maxdV"] = float((a[0] - b[0]).abs().max())
    r["iters_equal"] = bool(torch.equal(a[1], b[1]))
    r["resid_bitwise"] = bool(torch.equal(a[2], b[2]))
    r["resid_maxdiff"] = float((a[2] - b[2]).abs().max())
    r["sum_iters"] = int(b[1].sum())
    r["sched"] = {k: getattr(SparseOperator(m, "cuda:0").sub, k) for k in ("D", "NS", "NT", "NSL", "P", "smem_bytes")} \
        if SparseOperator(m, "cuda:0").sub is not None else None
    out[f"b{nb - 1}_tau{tau}"] = r
    print(json.dumps({f"b{nb - 1}_tau{tau}": r}), flush=True)

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 525600
spec = GenSpec(n_buses=5001, seed=0)
m = build_network(spec)
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
V = torch.empty_like(S)
it = torch.empty(tau, dtype=torch.int32, device="cuda:0")
rs = torch.empty(tau, dtype=torch.float64, device="cuda:0")
op = SparseOperator(m, "cuda:0")
ms = timed(lambda: op.solve(S, opts, V=V, iters=it, resid=rs), reps=2)
n = int(it.sum())
r = {"ms": ms, "sum_iters": n, "max_iters": int(it.max()), "alg_GBps": 48 * 5000 * n / ms / 1e6,
     "compulsory_GBps": 32 * 5000 * tau / ms / 1e6, "kernel": op.kernel, "resid_max": float(rs.max())}
print(json.dumps({"c3_full": r}), flush=True)

# case-major (F-order) S / V: each case's column is one contiguous 80 KB block (1-D bulk copies)
Sf = S.t().contiguous().t()
del S
torch.cuda.empty_cache()
Vf = torch.empty_like(Sf)
ms = timed(lambda: op.solve(Sf, opts, V=Vf, iters=it, resid=rs), reps=2)
r = {"ms": ms, "sum_iters": int(it.sum()), "alg_GBps": 48 * 5000 * n / ms / 1e6, "layout": "case-major"}
print(json.dumps({"c3_full_case_major": r}), flush=True)
