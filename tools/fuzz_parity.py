"""Randomised parity sweep (one-off check, not a unit test): random radial
feeders, batch sizes and load scales through every GPU path, against the
oracle's per-case restatement; then the same feeder with random tie branches
between demand buses (meshed: general sparse kernel, meshed ZIP kernel)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2403_04578_b200 import (Branch, GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,  # noqa: E402
                                   batch_solve_dense, batch_solve_sparse, build_network, gen_scenarios)
from oracle import tpf_oracle as orc  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bad = 0
t0 = time.time()
for trial in range(n_cases):
    nb = int(rng.choice([2, 3, 5, 9, 17, 33, 41, 57, 64, 65, 96, 101, 104, 105, 106, 150, 300]))
    kmax = int(rng.integers(1, 6))
    scale = float(rng.choice([0.3, 1.0, 3.0, 8.0]))
    spec = GenSpec(n_buses=nb, k_max=kmax, seed=int(rng.integers(0, 10_000)), load_scale=scale)
    model = build_network(spec)
    tau = int(rng.integers(1, 700))
    S = gen_scenarios(model, tau, spec).values.copy()
    if rng.random() < 0.3:
        S[:, rng.integers(0, tau)] = 0.0
    loads = LoadMatrix(S)
    opts = SolveOptions()
    y, src, vs = model.admittance.y_dd, model.source_injection(), model.slack.v_s
    V, n, mask, _ = orc.dense_per_case(y, src, vs, S, opts.tolerance, opts.max_iterations, opts.residual_tolerance)
    for name, fn in (("dense", lambda: batch_solve_dense(model, loads, opts)),
                     ("sparse", lambda: batch_solve_sparse(model, loads, opts)),
                     ("dense-pinned-chunks", lambda: batch_solve_dense(model, loads, opts, chunk_cases=37))):
        out = fn()
        dn = np.abs(out.iterations_per_case.astype(int) - n)
        good = mask & out.converged_mask
        dv = np.abs(out.values[:, good] - V[:, good]).max(initial=0.0)
        ok = dn.max(initial=0) <= 1 and np.array_equal(out.converged_mask, mask) and dv <= 1e-9 \
            and out.iterations == int(n.max(initial=0))
        if not ok:
            bad += 1
            print(f"MISMATCH {name} nb={nb} kmax={kmax} scale={scale} tau={tau}: max|dn|={dn.max()} "
                  f"mask_eq={np.array_equal(out.converged_mask, mask)} dv={dv:.2e} it={out.iterations}/{n.max()}")
    # ZIP on the same feeder
    w = rng.dirichlet([1.0, 1.0, 1.0], size=model.n_demand)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    zm = NetworkModel.from_branches(model.branches, nb, slack=model.slack, zip_coeffs=z)
    zo = batch_solve_dense(zm, loads, opts)  # tree kernel, or the thread-per-case kernel for deep feeders
    ZV, zn, zmask, _, zit = orc.dense_zip_batch(zm.admittance.y_dd, zm.source_injection(), vs, z.alpha_z,
                                                z.alpha_i, z.alpha_p, S)
    okz = np.array_equal(zo.iterations_per_case, zn) and np.array_equal(zo.converged_mask, zmask) and \
        np.abs(zo.values[:, zmask] - ZV[:, zmask]).max(initial=0) <= 1e-9
    if not okz:
        bad += 1
        print(f"MISMATCH zip nb={nb} tau={tau}: counts_eq={np.array_equal(zo.iterations_per_case, zn)} "
              f"mask_eq={np.array_equal(zo.converged_mask, zmask)}")
    # meshed: tie branches between demand buses
    if nb < 4:
        continue
    ties = list(model.branches)
    for _ in range(int(rng.integers(1, max(2, nb // 8)))):
        i, j = (int(x) for x in rng.choice(np.arange(1, nb), 2, replace=False))
        ties.append(Branch(from_bus=i, to_bus=j, r=float(rng.uniform(0.005, 0.05)), x=float(rng.uniform(0.005, 0.05))))
    mm = NetworkModel.from_branches(ties, nb, slack=model.slack)
    y, src = mm.admittance.y_dd, mm.source_injection()
    V, n, mask, _ = orc.dense_per_case(y, src, vs, S, opts.tolerance, opts.max_iterations, opts.residual_tolerance)
    for name, fn in (("mesh-dense", lambda: batch_solve_dense(mm, loads, opts)),
                     ("mesh-sparse", lambda: batch_solve_sparse(mm, loads, opts))):
        out = fn()
        dn = np.abs(out.iterations_per_case.astype(int) - n)
        good = mask & out.converged_mask
        dv = np.abs(out.values[:, good] - V[:, good]).max(initial=0.0)
        if not (dn.max(initial=0) <= 1 and np.array_equal(out.converged_mask, mask) and dv <= 1e-9):
            bad += 1
            print(f"MISMATCH {name} nb={nb} tau={tau}: max|dn|={dn.max()} "
                  f"mask_eq={np.array_equal(out.converged_mask, mask)} dv={dv:.2e}")
    zmm = NetworkModel.from_branches(ties, nb, slack=model.slack, zip_coeffs=z)
    zo = batch_solve_dense(zmm, loads, opts)
    ZV, zn, zmask, _, zit = orc.dense_zip_batch(y, src, vs, z.alpha_z, z.alpha_i, z.alpha_p, S)
    dn = np.abs(zo.iterations_per_case.astype(int) - zn)
    if not (dn.max(initial=0) <= 1 and np.array_equal(zo.converged_mask, zmask) and
            np.abs(zo.values[:, zmask] - ZV[:, zmask]).max(initial=0) <= 1e-9):
        bad += 1
        print(f"MISMATCH mesh-zip nb={nb} tau={tau}: max|dn|={dn.max()} "
              f"mask_eq={np.array_equal(zo.converged_mask, zmask)}")
print(f"{n_cases} trials, {bad} mismatches, {time.time() - t0:.0f}s")
