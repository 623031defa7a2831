"""Meshed ZIP at C2 size (b=100, tau=525,600): the per-case fixed-pattern LU
kernel (tpf_sparse_zip_lu_c128), and the same kernel against the radial
chain kernel on the radial feeder (what a fill-free pattern costs)."""
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import (Branch, GenSpec, LoadMatrix, NetworkModel, SolveOptions,  # noqa: E402
                                   ZipCoefficients, build_network, gen_scenarios)
from paper_2403_04578_b200 import dense as dn  # noqa: E402
from paper_2403_04578_b200._device import ModelContract, loads_to_device  # noqa: E402
from paper_2403_04578_b200.sparse import zip_lu_schedule  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 525_600
for nbus, loops in ((101, 0), (101, 10), (101, 30)):
    spec = GenSpec(n_buses=nbus, seed=0)
    base = build_network(spec)
    b = base.n_demand
    rng = np.random.default_rng(5)
    branches = list(base.branches)
    for _ in range(loops):
        i, j = (int(x) for x in rng.choice(np.arange(1, nbus), 2, replace=False))
        branches.append(Branch(from_bus=i, to_bus=j, r=0.02, x=0.03))
    w = rng.dirichlet([1.0, 1.0, 1.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(branches, nbus, slack=base.slack, zip_coeffs=z)
    loads = LoadMatrix(gen_scenarios(model, tau, spec).values)
    dev = torch.device("cuda:0")
    S = SimpleNamespace(values=loads_to_device(loads.values, dev))
    c = ModelContract.of(model)
    sch = zip_lu_schedule(c.y_dd)
    runs = [("lu", lambda: dn._solve_zip_lu(model, c, S, SolveOptions(), None, True))]
    if loops == 0:
        runs.append(("chain", lambda: dn._solve_zip_chain(model, c, S, SolveOptions(), None, True)))
    res = {}
    for name, fn in runs:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0, out)
    lu = res["lu"][1]
    sum_n = int(lu.iterations_per_case.sum().item())
    line = "b=%d loops=%d nslot=%d fill=%d: lu %.1f ms (device-resident loads), sum_n %d, converged %d/%d" % (
        b, loops, sch.nslot, sch.fill, 1e3 * res["lu"][0], sum_n, int(lu.converged_mask.sum().item()), tau)
    if "chain" in res:
        ch = res["chain"][1]
        line += "; chain %.1f ms, counts equal %s, max|dV| %.1e" % (
            1e3 * res["chain"][0], torch.equal(ch.iterations_per_case, lu.iterations_per_case),
            (ch.values - lu.values).abs().max().item())
    print(line, flush=True)
