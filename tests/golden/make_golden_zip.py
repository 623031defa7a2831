"""ZIP-load fixtures from the REFERENCE (dense.py:214-230 -> fpi.py:107-206).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_zip.py

For each fixture: a radial feeder from the reference generator with mixed
Z/I/P fractions per node (seeded), a load batch (some zero-load cases and, for
``zip9_heavy``, an infeasible one), and the reference batch_solve_dense result
(which loops fpi_solve per case) plus per-case iterations / step flags from
fpi_solve itself.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from tpflow import (GenSpec, LoadMatrix, NetworkModel, SolveOptions, batch_solve_dense,  # noqa: E402
                    build_network, fpi_solve, gen_scenarios)
from tpflow.network import ZipCoefficients  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "zip")


def zip_model(n_buses, seed, kind):
    base = build_network(GenSpec(n_buses=n_buses, seed=seed))
    b = base.n_demand
    rng = np.random.default_rng(100 + seed)
    if kind == "mixed":
        w = rng.dirichlet([1.0, 1.0, 1.0], size=b)
    elif kind == "pure_zi":  # alpha_p = 0 everywhere: one application per case
        w = np.stack([rng.uniform(0, 1, b), np.zeros(b), np.zeros(b)], axis=1)
        w[:, 1] = 1.0 - w[:, 0]
    else:
        raise ValueError(kind)
    w = w / w.sum(axis=1, keepdims=True)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    return NetworkModel.from_branches(base.branches, n_buses, slack=base.slack, zip_coeffs=z), z


def save(name, n_buses, seed, tau, kind="mixed", scale=1.0, heavy=False, opts=SolveOptions()):
    model, z = zip_model(n_buses, seed, kind)
    S = gen_scenarios(model, tau, GenSpec(n_buses=n_buses, seed=seed, load_scale=scale)).values.copy()
    S[:, 1] = 0.0  # a zero-load case
    if heavy:
        S[:, 2] *= 400.0  # infeasible
    r = batch_solve_dense(model, LoadMatrix(S), opts)
    n, met = [], []
    for j in range(tau):
        res = fpi_solve(model, S[:, j], opts)
        n.append(res.iterations)
        met.append(bool(res.step_inf.size and res.step_inf[-1] < opts.tolerance) or res.iterations == 1)
    y = model.admittance.y_dd.tocsc()
    np.savez(os.path.join(HERE, name + ".npz"), n_buses=n_buses, seed=seed, kind=kind,
             alpha_z=z.alpha_z, alpha_i=z.alpha_i, alpha_p=z.alpha_p, S=S,
             ydd_data=y.data, ydd_indices=y.indices, ydd_indptr=y.indptr, src=model.source_injection(),
             V=r.values, iterations=r.iterations, mask=r.converged_mask, residuals=r.residuals,
             n_case=np.array(n), tol=opts.tolerance, max_iter=opts.max_iterations,
             residual_tol=opts.residual_tolerance)
    print(name, "iterations", r.iterations, "converged", int(r.converged_mask.sum()), "/", tau, file=sys.stderr)


save("zip9_mixed", 9, 0, 40)
save("zip9_heavy", 9, 1, 20, heavy=True)
save("zip9_pure_zi", 9, 2, 20, kind="pure_zi")
save("zip101_mixed", 101, 0, 64, scale=3.0)
