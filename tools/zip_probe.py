"""ZIP loads at C2 scale: GPU (one launch, per-case factorization on chip) vs the
reference's per-case route (oracle restatement, timed on a sample)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import (GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,  # noqa: E402
                                   batch_solve_dense, build_network, gen_scenarios)
from paper_2403_04578_b200.dense import solve_zip  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import tpf_oracle as orc  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 525600
spec = GenSpec(n_buses=101, seed=0)
base = build_network(spec)
b = base.n_demand
w = np.random.default_rng(0).dirichlet([1.0, 1.0, 1.0], size=b)
z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
model = NetworkModel.from_branches(base.branches, 101, slack=base.slack, zip_coeffs=z)
S = gen_scenarios(model, tau, spec).values
loads = LoadMatrix(torch.from_numpy(S).pin_memory().numpy())
out = solve_zip(model, loads, SolveOptions(), return_on_device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
out = solve_zip(model, loads, SolveOptions(), return_on_device=True)
torch.cuda.synchronize()
gpu_s = time.perf_counter() - t0
n = 300
t0 = time.perf_counter()
orc.dense_zip_batch(model.admittance.y_dd, model.source_injection(), model.slack.v_s, z.alpha_z, z.alpha_i,
                    z.alpha_p, S[:, :n])
cpu_per_case = (time.perf_counter() - t0) / n
print(json.dumps({"tau": tau, "b": b, "gpu_seconds_incl_h2d": gpu_s, "gpu_pf_per_s": tau / gpu_s,
                  "sum_iterations": int(out.iterations_per_case.sum()), "batch_iterations": out.iterations,
                  "converged": int(out.converged_mask.sum()),
                  "cpu_reference_route_pf_per_s_1_core": 1.0 / cpu_per_case, "cpu_sample_cases": n}))
