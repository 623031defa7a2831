"""Generate the golden fixtures by running the REFERENCE `tpflow` itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each fixture ``<name>.npz`` holds the network contract (Y_dd as CSC arrays,
src = Y_ds v_s, v_s), the load matrix S (b x tau) and the reference outputs
of ``batch_solve_dense`` / ``batch_solve_sparse`` (V, iterations,
converged_mask, residuals), plus per-case iteration counts from the reference's
own single-case solver ``fpi_solve`` where tau is small enough.  Large configs
are stored as column slices: the slice is solved as its own batch by the
reference, so the fixture is self-consistent.  Versions of numpy/scipy are
recorded in ``manifest.json``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import scipy

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import tpflow  # noqa: E402
from tpflow import (GenSpec, LoadMatrix, NetworkModel, SlackSpec, Branch,  # noqa: E402
                    SolveOptions, batch_solve_dense, batch_solve_sparse,
                    build_network, fpi_solve, gen_scenarios)

HERE = os.path.dirname(os.path.abspath(__file__))


def model_arrays(model):
    y = model.admittance.y_dd.tocsc()
    return dict(ydd_data=y.data, ydd_indices=y.indices.astype(np.int64),
                ydd_indptr=y.indptr.astype(np.int64), ydd_shape=np.array(y.shape),
                src=model.source_injection(), v_s=np.array(model.slack.v_s))


def save(name, model, S, dense=True, sparse=True, per_case=False, opts=SolveOptions(),
         extra=None):
    out = dict(model_arrays(model), S=S, tol=opts.tolerance, max_iter=opts.max_iterations,
               residual_tol=opts.residual_tolerance)
    loads = LoadMatrix(S)
    if dense:
        r = batch_solve_dense(model, loads, opts)
        out.update(dense_V=r.values, dense_iterations=r.iterations,
                   dense_mask=r.converged_mask, dense_residuals=r.residuals)
    if sparse:
        r = batch_solve_sparse(model, loads, opts)
        out.update(sparse_V=r.values, sparse_iterations=r.iterations,
                   sparse_mask=r.converged_mask, sparse_residuals=r.residuals)
    if per_case:
        n = []
        vs = []
        for j in range(S.shape[1]):
            res = fpi_solve(model, S[:, j], opts)
            n.append(res.iterations)
            vs.append(res.v)
        out.update(fpi_iterations=np.array(n, dtype=np.int32), fpi_V=np.stack(vs, axis=1))
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, S.shape, {k: v for k, v in out.items() if k.endswith("iterations") and np.ndim(v) == 0})


def two_bus(z, v0=1.0):
    z = complex(z)
    return NetworkModel.from_branches([Branch(0, 1, z.real, z.imag)], 2, slack=SlackSpec(complex(v0)))


def feasible(model, tau, seed, scale=1.0):
    return gen_scenarios(model, tau, GenSpec(n_buses=model.n_demand + 1, seed=seed,
                                             load_scale=scale)).values


def hardest_columns(model, S, k):
    """Indices of the k columns with the largest single-case iteration counts."""
    from scipy.sparse.linalg import splu
    lu = splu(model.admittance.y_dd.tocsc())
    K = -lu.solve(np.eye(model.n_demand, dtype=complex))
    W = K @ model.source_injection()
    b, tau = S.shape
    v = np.full((b, tau), abs(model.slack.v_s) + 0j)
    n = np.zeros(tau, dtype=int)
    active = np.ones(tau, dtype=bool)
    for it in range(100):
        idx = np.where(active)[0]
        if idx.size == 0:
            break
        vn = K @ (np.conj(S[:, idx]) / np.conj(v[:, idx])) + W[:, None]
        d = np.abs(vn - v[:, idx]).max(axis=0)
        v[:, idx] = vn
        n[idx] += 1
        active[idx[d < 1e-10]] = False
    return np.argsort(-n, kind="stable")[:k], n


def main():
    manifest = dict(numpy=np.__version__, scipy=scipy.__version__, tpflow=tpflow.__version__,
                    python=sys.version.split()[0], fixtures={})
    nine = build_network(GenSpec(n_buses=9, seed=42))

    # known answer: two-bus V_HIGH = (1 + sqrt(0.96))/2 (test_dense.py:114-116)
    save("twobus_known", two_bus(0.1), np.array([[0.1 + 0j]]))
    # divergence as data (test_dense.py:81-87, 104-112)
    save("twobus_infeasible", two_bus(1.0 + 0.5j),
         np.array([[0.05 + 0.02j, 3.0 + 2.0j, 0.18 + 0.11j, 0.01 + 0j]]))
    # batch == per case (test_dense.py:62-79)
    save("nine_t500", nine, feasible(nine, 500, 21), per_case=True)
    # zero-load rows (test_sparse.py:154-162)
    z = feasible(nine, 12, 39).copy()
    z[0, :] = 0.0
    z[4, 6] = 0.0
    save("nine_zero_rows", nine, z)
    # zero-load batch: <= 1 iteration (test_dense.py:140-144)
    save("nine_zero_batch", nine, np.zeros((8, 6), dtype=complex))
    # iterate sequences at fixed caps (test_sparse.py:170-180)
    caps = feasible(nine, 8, 41)
    for cap in (1, 2, 3, 5, 8):
        save(f"nine_cap{cap}", nine, caps,
             opts=SolveOptions(tolerance=1e-16, max_iterations=cap, residual_tolerance=np.inf))
    # acceptance criterion 3 (test_acceptance.py:90-108)
    spec = GenSpec(n_buses=101, seed=6)
    m101 = build_network(spec)
    save("acc3_b100_t100", m101, gen_scenarios(m101, 100, spec).values)
    # acceptance criterion 7 mixed zero loads (test_acceptance.py:235-245)
    spec13 = GenSpec(n_buses=13, seed=99)
    m13 = build_network(spec13)
    vals = gen_scenarios(m13, 40, spec13).values.copy()
    vals[1, :] = 0.0
    vals[5, ::3] = 0.0
    save("acc7_mixed_zero", m13, vals)
    # asymmetric matrix-supplied Y_dd (test_fpi.py:200-215)
    rng = np.random.default_rng(18)
    n = 6
    y_dd = rng.normal(0, 1, (n, n)) + 1j * rng.normal(0, 1, (n, n))
    np.fill_diagonal(y_dd, 0)
    np.fill_diagonal(y_dd, np.abs(y_dd).sum(axis=1) + 20.0)
    y_ds = -(y_dd @ np.ones(n))[:, None]
    masym = NetworkModel.from_admittance(y_dd, y_ds)
    s = 0.01 * (rng.uniform(0.5, 1, n) + 0.3j * rng.uniform(0, 1, n))
    save("asym6", masym, np.stack([s, 2 * s, 0.5 * s], axis=1), per_case=True)

    # C1: GenSpec(35, seed=0), tau = 8760; slice of 512 columns (generated at full tau)
    spec1 = GenSpec(n_buses=35, seed=0)
    m1 = build_network(spec1)
    S1 = gen_scenarios(m1, 8760, spec1).values
    save("c1_slice512", m1, np.ascontiguousarray(S1[:, :512]), per_case=True)
    # C2: GenSpec(101, seed=0), tau = 525,600; 192 columns: hardest 64 + first 128
    spec2 = GenSpec(n_buses=101, seed=0)
    m2 = build_network(spec2)
    S2 = gen_scenarios(m2, 525600, spec2).values
    hard, n2 = hardest_columns(m2, S2, 64)
    cols = np.concatenate([hard, np.arange(128)])
    save("c2_slice192", m2, np.ascontiguousarray(S2[:, cols]), per_case=True,
         extra=dict(columns=cols, c2_sum_n=int(n2.sum()), c2_max_n=int(n2.max()),
                    c2_hist=np.bincount(n2)))
    del S2
    # C5: GenSpec(1001, seed=0, load_scale=21), tau = 8760; hardest 16 + first 16
    spec5 = GenSpec(n_buses=1001, seed=0, load_scale=21)
    m5 = build_network(spec5)
    S5 = gen_scenarios(m5, 8760, spec5).values
    hard5, n5 = hardest_columns(m5, S5, 16)
    cols5 = np.concatenate([hard5, np.arange(16)])
    save("c5_slice32", m5, np.ascontiguousarray(S5[:, cols5]), sparse=False,
         extra=dict(columns=cols5, c5_sum_n=int(n5.sum()), c5_max_n=int(n5.max())))
    # C3: GenSpec(5001, seed=0), sparse; 6 columns of a tau=600 batch
    spec3 = GenSpec(n_buses=5001, seed=0)
    m3 = build_network(spec3)
    S3 = gen_scenarios(m3, 600, spec3).values
    save("c3_slice6", m3, np.ascontiguousarray(S3[:, :6]), dense=False)

    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            manifest["fixtures"][f] = os.path.getsize(os.path.join(HERE, f))
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
