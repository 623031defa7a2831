"""ZIP at C2 size: tree kernel (one case per SM) vs the thread-per-case chain kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import (GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,  # noqa: E402
                                   build_network, gen_scenarios)
from paper_2403_04578_b200 import dense as dn  # noqa: E402
from paper_2403_04578_b200._device import ModelContract  # noqa: E402

for nbus, tau in ((201, 131072), (301, 131072), (501, 65536)):
    spec = GenSpec(n_buses=nbus, seed=0)
    base = build_network(spec)
    b = base.n_demand
    w = np.random.default_rng(0).dirichlet([1.0, 1.0, 1.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(base.branches, nbus, slack=base.slack, zip_coeffs=z)
    loads = LoadMatrix(gen_scenarios(model, tau, spec).values)
    c = ModelContract.of(model)
    res = {}
    for name, fn in (("tree", lambda: dn.solve_zip(model, loads, SolveOptions(), return_on_device=True)),
                     ("chain", lambda: dn._solve_zip_chain(model, c, loads, SolveOptions(), None, True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0, out)
    same = torch.equal(res["tree"][1].iterations_per_case, res["chain"][1].iterations_per_case)
    dv = (res["tree"][1].values - res["chain"][1].values).abs().max().item()
    print("b=%d tau=%d: tree %.1f ms, chain %.1f ms (incl. H2D); counts equal %s, max|dV| %.1e" % (
        b, tau, 1e3 * res["tree"][0], 1e3 * res["chain"][0], same, dv))
