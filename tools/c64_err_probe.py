"""complex64 twins vs the complex128 engine at the reference tolerance (1e-10).

max |V_c64 - V_c128| over the full C2 batch (b=100, tau=525,600) for the dense
twin, and over a C2 slice for the sparse twin, at several c64 tolerances.
Usage: python tools/c64_err_probe.py [tau]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator, SparseOperator, SolveOptions  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 525600
spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
ref, it_ref = DenseOperator(m, "cuda:0").solve(S, SolveOptions())
S32 = S.to(torch.complex64)
out = {"tau": tau}
for tol in (1e-6, 1e-7):
    for name, op in (("dense", DenseOperator(m, "cuda:0", dtype=np.complex64)),
                     ("sparse", SparseOperator(m, "cuda:0", dtype=np.complex64))):
        n = tau if name == "dense" else min(tau, 65536)
        V, it = op.solve(S32[:, :n], SolveOptions(tolerance=tol))
        d = (V.to(torch.complex128) - ref[:, :n]).abs()
        out[f"{name}_tol{tol:g}"] = {"max_abs_err": float(d.max()), "p99_case_max": float(torch.quantile(d.max(0).values[:65536], 0.99)),
                                    "mean_it": float(it.double().mean()), "max_it": int(it.max()),
                                    "ref_mean_it": float(it_ref[:n].double().mean())}
print(json.dumps(out, indent=1))
