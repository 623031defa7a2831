"""ZIP-load fixtures from the REFERENCE (dense.py:214-230 -> fpi.py:107-206).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_zip.py [names...]

For each fixture: a radial feeder (``*_mesh``: plus tie branches closing loops
among the demand buses, the reference's meshed per-case SuperLU route) from the reference generator with mixed
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
from tpflow.network import Branch, ZipCoefficients  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "zip")


def zip_model(n_buses, seed, kind, loops=0):
    base = build_network(GenSpec(n_buses=n_buses, seed=seed))
    branches = list(base.branches)
    if loops:  # tie branches between demand buses close loops: a meshed Y_dd
        rng_l = np.random.default_rng(200 + seed)
        linked = {frozenset((br.from_bus, br.to_bus)) for br in branches}
        while loops:
            i, j = (int(x) for x in rng_l.choice(np.arange(1, n_buses), 2, replace=False))
            if frozenset((i, j)) in linked:
                continue
            linked.add(frozenset((i, j)))
            loops -= 1
            br = branches[int(rng_l.integers(len(branches)))]
            branches.append(Branch(from_bus=i, to_bus=j, r=br.r * 2.0, x=br.x * 2.0))
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
    return NetworkModel.from_branches(branches, n_buses, slack=base.slack, zip_coeffs=z), z


def save(name, n_buses, seed, tau, kind="mixed", scale=1.0, heavy=False, opts=SolveOptions(), loops=0,
         warm=False):
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        return
    model, z = zip_model(n_buses, seed, kind, loops)
    if warm:  # opts.initial_voltage: a seeded non-flat start (fpi.py:141-145)
        rng_w = np.random.default_rng(300 + seed)
        b = model.n_demand
        v0 = rng_w.uniform(0.9, 1.05, b) * np.exp(1j * rng_w.uniform(-0.05, 0.05, b))
        opts = SolveOptions(tolerance=opts.tolerance, max_iterations=opts.max_iterations,
                            residual_tolerance=opts.residual_tolerance, initial_voltage=v0)
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
             residual_tol=opts.residual_tolerance,
             **({} if opts.initial_voltage is None else {"initial_voltage": opts.initial_voltage}))
    print(name, "iterations", r.iterations, "converged", int(r.converged_mask.sum()), "/", tau, file=sys.stderr)


save("zip9_mixed", 9, 0, 40)
save("zip9_heavy", 9, 1, 20, heavy=True)
save("zip9_pure_zi", 9, 2, 20, kind="pure_zi")
save("zip101_mixed", 101, 0, 64, scale=3.0)
save("zip9_mesh", 9, 3, 24, loops=4)
save("zip101_mesh", 101, 4, 48, scale=2.0, loops=8)
# warm starts (opts.initial_voltage) on each GPU route: chain (b <= 384), tree (b > 384), meshed LU
save("zip9_warm", 9, 5, 24, warm=True)
save("zip501_warm", 501, 6, 12, scale=2.0, warm=True)
save("zip9_mesh_warm", 9, 7, 24, loops=4, warm=True)
