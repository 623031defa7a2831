"""Host-side logic of the boundary: types, validation, LU preparation.

All CPU; no kernels are launched."""

import numpy as np
import pytest
from scipy import sparse

from paper_2403_04578_b200 import (GenSpec, LoadMatrix, PowerTensor, SingularSystemError,
                                   SolveOptions, VoltageBatch, build_network, factorize_ydd,
                                   reshape_tensor, unreshape, batch_solve_dense, batch_solve_sparse,
                                   solve_batch, NetworkModel, ZipCoefficients, MemoryGuardError)
from paper_2403_04578_b200.sparse import leaf_first_order, lu_solve_host


class TestTypes:
    def test_fig4_layout(self):
        # test_dense.py:21-35: case (i,j,k) lands in column i*6 + j*3 + k
        rng = np.random.default_rng(0)
        t = PowerTensor(rng.standard_normal((2, 2, 3, 3)) * (1 + 1j))
        loads = reshape_tensor(t)
        assert loads.values.shape == (3, 12)
        for i in range(2):
            for j in range(2):
                for k in range(3):
                    assert np.array_equal(loads.values[:, i * 6 + j * 3 + k], t.values[i, j, k, :])

    def test_round_trip(self):
        rng = np.random.default_rng(1)
        t = PowerTensor(rng.standard_normal((4, 2, 5, 6)) + 1j * rng.standard_normal((4, 2, 5, 6)))
        back = unreshape(reshape_tensor(t))
        assert np.array_equal(back.values, t.values) and back.dims == t.dims

    def test_options_validation(self):
        with pytest.raises(ValueError):
            SolveOptions(tolerance=0)
        with pytest.raises(ValueError):
            SolveOptions(max_iterations=0)

    def test_voltage_batch_accessors(self):
        vb = VoltageBatch(values=np.array([[0.5 + 0.5j, 1.0 + 0j]]), iterations=3,
                          converged_mask=np.array([True, True]), residuals=np.zeros(2))
        assert vb.tau == 2
        assert vb.magnitudes()[0, 0] == pytest.approx(np.sqrt(0.5))
        assert vb.angles()[0, 0] == pytest.approx(np.pi / 4)


class TestBoundaryErrors:
    """Errors the reference raises before any arithmetic (dense.py:143-148, sparse.py:121-136)."""

    def test_row_count_mismatch(self):
        m = build_network(GenSpec(n_buses=9, seed=42))
        with pytest.raises(ValueError, match="rows"):
            batch_solve_dense(m, LoadMatrix([[0.1 + 0j]]))
        with pytest.raises(ValueError, match="rows"):
            batch_solve_sparse(m, LoadMatrix([[0.1 + 0j]]))

    def test_zip_models(self):
        m = build_network(GenSpec(n_buses=9, seed=42))
        b = m.n_demand
        zm = NetworkModel(admittance=m.admittance, slack=m.slack,
                          zip=ZipCoefficients(np.full(b, 0.2), np.full(b, 0.1), np.full(b, 0.7)))
        loads = LoadMatrix(np.full((b, 2), 0.01 + 0j))
        # radial ZIP models run on the GPU (tests/test_zip_gpu.py); here: no CPU fallback
        with pytest.raises(RuntimeError, match="CUDA device"):
            batch_solve_dense(zm, loads)
        with pytest.raises(ValueError, match="constant-power"):
            batch_solve_sparse(zm, loads)
        # a meshed network with ZIP loads: the per-case LU kernel (tests/test_zip_gpu.py), no CPU fallback
        from scipy import sparse as sp
        y = m.admittance.y_dd.tolil()
        dense = m.admittance.y_dd.toarray()
        # a node, a neighbour and that neighbour's other neighbour: closing the triangle
        # makes a cycle among the demand nodes (Y_dd is no longer a forest)
        i, j = next((i, j) for i in range(b) for k in range(b) for j in range(b)
                    if len({i, j, k}) == 3 and dense[i, k] != 0 and dense[k, j] != 0 and dense[i, j] == 0)
        y[i, j] = y[j, i] = -1.0 + 1.0j
        mesh = NetworkModel.from_admittance(sp.csc_matrix(y), m.admittance.y_ds, slack=m.slack,
                                            zip_coeffs=zm.zip)
        with pytest.raises(RuntimeError, match="CUDA device"):
            batch_solve_dense(mesh, loads)
        # its fixed-pattern schedule (sparse.zip_lu_schedule) solves B x = r like SuperLU
        from paper_2403_04578_b200.sparse import zip_lu_schedule, zip_lu_solve_host
        sch = zip_lu_schedule(mesh.admittance.y_dd)
        assert sch.fill > 0 and sorted(sch.orig.tolist()) == list(range(b))
        rng = np.random.default_rng(1)
        d = 0.2 * rng.normal(size=b) - 0.1j
        r = rng.normal(size=b) + 1j * rng.normal(size=b)
        ref = sp.linalg.spsolve((mesh.admittance.y_dd + sp.diags(d)).tocsc(), r)
        assert np.abs(zip_lu_solve_host(sch, d, r) - ref).max() <= 1e-12 * np.abs(ref).max()

    def test_memory_guard(self):
        m = build_network(GenSpec(n_buses=9, seed=42))
        loads = LoadMatrix(np.full((8, 50), 0.01 + 0j))
        with pytest.raises(MemoryGuardError, match="chunk"):
            batch_solve_sparse(m, loads, max_nnz=100)

    def test_dispatcher(self):
        m = build_network(GenSpec(n_buses=9, seed=42))
        with pytest.raises(ValueError, match="unknown method"):
            solve_batch("bogus", m, LoadMatrix(np.zeros((8, 1), complex)))
        with pytest.raises(NotImplementedError):
            solve_batch("nr", m, LoadMatrix(np.zeros((8, 1), complex)))


class TestTreeLU:
    @pytest.mark.parametrize("n_buses", [2, 9, 101, 1001])
    def test_leaf_first_lu_has_no_fill_and_solves(self, n_buses):
        m = build_network(GenSpec(n_buses=n_buses, seed=3))
        y = m.admittance.y_dd
        f = factorize_ydd(y)
        b = m.n_demand
        assert f.ordering == "leaf-first"
        # zero fill: strictly-lower + strictly-upper entries == off-diagonals of Y_dd
        assert f.l_col.size + f.u_col.size == y.nnz - b
        rng = np.random.default_rng(n_buses)
        r = rng.standard_normal(b) + 1j * rng.standard_normal(b)
        x = lu_solve_host(f, r)
        assert np.abs(y @ x - r).max() / np.abs(r).max() < 1e-12

    def test_general_matrix_uses_colamd_with_pivoting(self):
        rng = np.random.default_rng(18)
        n = 6
        y = rng.normal(0, 1, (n, n)) + 1j * rng.normal(0, 1, (n, n))
        np.fill_diagonal(y, 0)
        np.fill_diagonal(y, np.abs(y).sum(axis=1) + 20.0)
        f = factorize_ydd(sparse.csc_matrix(y))
        assert f.ordering == "colamd"
        r = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        assert np.abs(y @ lu_solve_host(f, r) - r).max() < 1e-12

    def test_singular_names_location(self):
        with pytest.raises(SingularSystemError, match=r"rows \[1\]"):
            factorize_ydd(sparse.csc_matrix(np.array([[1.0, 0.0], [0.0, 0.0]])))

    def test_leaf_first_detects_cycles(self):
        y = sparse.csr_matrix(np.ones((3, 3)) + 2 * np.eye(3))
        assert leaf_first_order(y) is None


class TestTreeSchedule:
    @pytest.mark.parametrize("n_buses", [2, 9, 101, 1001])
    def test_schedule_sweeps_solve_ydd(self, n_buses):
        from paper_2403_04578_b200.sparse import tree_schedule, tree_solve_host
        m = build_network(GenSpec(n_buses=n_buses, seed=5))
        t = tree_schedule(factorize_ydd(m.admittance.y_dd), m.source_injection())
        assert t is not None
        b = m.n_demand
        rng = np.random.default_rng(n_buses)
        r = rng.standard_normal(b) + 1j * rng.standard_normal(b)
        x = tree_solve_host(t, r)
        assert np.abs(m.admittance.y_dd @ x - r).max() / np.abs(r).max() < 1e-12
        # children contiguous, parents one level up, slots within the TMEM budget
        info = t.node_info.reshape(b, 4)
        offs = t.level_info[:t.levels + 1]
        for d in range(1, t.levels):
            for mm in range(offs[d], offs[d + 1]):
                p = info[mm, 1]
                assert offs[d - 1] <= p < offs[d]
                assert info[p, 2] <= mm < info[p, 2] + info[p, 3]
        assert t.slots <= 16

    @pytest.mark.parametrize("n_buses", [2, 9, 1001])
    def test_ell_rows_reproduce_ydd_in_level_order(self, n_buses):
        """tpf_sparse_tree_build_ell (host helper of the fused residual) == Y_dd permuted to level order."""
        from paper_2403_04578_b200.sparse import tree_schedule, tree_ell
        from paper_2403_04578_b200._device import ModelContract
        m = build_network(GenSpec(n_buses=n_buses, seed=7))
        t = tree_schedule(factorize_ydd(m.admittance.y_dd), m.source_injection())
        w, col, val = tree_ell(t, ModelContract.of(m))
        b = m.n_demand
        y = m.admittance.y_dd.toarray()
        orig = t.node_info.reshape(b, 4)[:, 0]
        dense = np.zeros((b, b), dtype=complex)
        col, val = col.reshape(w, b), val.reshape(w, b)
        for mm in range(b):
            row = m.admittance.y_dd.getrow(orig[mm])
            n = row.nnz
            assert (col[n:, mm] == -1).all() and (val[n:, mm] == 0).all()
            # same entries in the same (original CSR) order
            assert np.array_equal(orig[col[:n, mm]], row.indices) and np.array_equal(val[:n, mm], row.data)
            dense[mm, col[:n, mm]] = val[:n, mm]
        assert np.array_equal(dense, y[np.ix_(orig, orig)])

    def test_c3_feeder_fits_the_tmem_budget(self):
        from paper_2403_04578_b200.sparse import tree_schedule
        m = build_network(GenSpec(n_buses=5001, seed=0))
        t = tree_schedule(factorize_ydd(m.admittance.y_dd), m.source_injection())
        assert t is not None and t.levels == 7 and t.slots == 16

    def test_general_matrix_has_no_tree_schedule(self):
        from paper_2403_04578_b200.sparse import tree_schedule
        rng = np.random.default_rng(18)
        y = rng.normal(0, 1, (6, 6)) + 1j * rng.normal(0, 1, (6, 6))
        np.fill_diagonal(y, np.abs(y).sum(axis=1) + 20.0)
        assert tree_schedule(factorize_ydd(sparse.csc_matrix(y)), np.zeros(6, complex)) is None


class TestDenseOperatorCache:
    def test_cache_returns_same_bits_and_tracks_content(self):
        from paper_2403_04578_b200.dense import dense_kw
        from paper_2403_04578_b200._device import ModelContract
        m = build_network(GenSpec(n_buses=30, seed=2))
        c = ModelContract.of(m)
        K1, W1 = dense_kw(c)
        K2, W2 = dense_kw(ModelContract.of(m))
        assert K1 is K2 and W1 is W2
        assert np.array_equal(K1, -np.linalg.inv(c.y_dd.toarray()))
        # a different feeder (or changed impedances) never hits the entry
        m2 = build_network(GenSpec(n_buses=30, seed=3))
        K3, _ = dense_kw(ModelContract.of(m2))
        assert K3 is not K1 and not np.array_equal(K3, K1)

    def test_singular_ydd_still_raises(self):
        from scipy import sparse as sp
        from paper_2403_04578_b200.dense import dense_kw
        from paper_2403_04578_b200._device import ModelContract
        c = ModelContract(b=2, y_dd=sp.csr_matrix(np.array([[1, 1], [1, 1]], dtype=complex)),
                          src=np.zeros(2, dtype=complex), v_s=1 + 0j, constant_power=True)
        with pytest.raises(np.linalg.LinAlgError):
            dense_kw(c)


class TestCaseSlices:
    @pytest.mark.parametrize("tau,parts", [(0, 1), (1, 3), (7, 3), (525600, 8), (10, 10)])
    def test_contiguous_cover(self, tau, parts):
        from paper_2403_04578_b200._device import case_slices
        sl = case_slices(tau, parts)
        assert len(sl) == parts and sl[0][0] == 0 and sl[-1][1] == tau
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        sizes = [hi - lo for lo, hi in sl]
        assert max(sizes) - min(sizes) <= 1


def test_engine_dtype_validation():
    from paper_2403_04578_b200._device import engine_dtype
    assert engine_dtype(None) == np.complex128
    assert engine_dtype(np.complex64) == np.complex64
    assert engine_dtype("complex64") == np.complex64
    with pytest.raises(ValueError):
        engine_dtype(np.float32)


def test_reference_model_objects_are_accepted_as_is():
    """A real tpflow.NetworkModel reduces to the same hot-path contract (skipped where the
    reference is not importable, e.g. on the GPU box)."""
    import os
    import sys
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    old = sys.dont_write_bytecode
    sys.dont_write_bytecode = True  # never write into the read-only reference tree
    try:
        import tpflow
    except Exception:  # pragma: no cover
        pytest.skip("reference not importable")
    finally:
        sys.path.remove(ref)
        sys.dont_write_bytecode = old
    from paper_2403_04578_b200._device import ModelContract
    spec_r = tpflow.GenSpec(n_buses=30, seed=3)
    mine = ModelContract.of(build_network(GenSpec(n_buses=30, seed=3)))
    theirs = ModelContract.of(tpflow.build_network(spec_r))
    assert (mine.y_dd != theirs.y_dd).nnz == 0
    assert np.array_equal(mine.src, theirs.src) and mine.v_s == theirs.v_s
    assert theirs.constant_power


def test_as_load_matrix_complex64_passthrough():
    """complex64 arrays reach the c64 twin as is; everything else becomes the
    reference's complex128 LoadMatrix (dense.py:57-78)."""
    import numpy as np
    from paper_2403_04578_b200 import LoadMatrix
    from paper_2403_04578_b200.dense import as_load_matrix
    a64 = (np.arange(12, dtype=np.float32).reshape(3, 4) * (1 + 1j)).astype(np.complex64)
    lm = as_load_matrix(a64, np.complex64)
    assert lm.values is a64 and lm.n_demand == 3 and lm.tau == 4 and lm.dims == (4,)
    assert as_load_matrix(a64).values.dtype == np.complex128  # c128 engine: the reference's conversion
    assert as_load_matrix(a64.astype(np.complex128), np.complex64).values.dtype == np.complex128
    ref = LoadMatrix(a64)
    assert as_load_matrix(ref, np.complex64) is ref


def test_zip_initial_voltage_length_checked_like_fpi_solve():
    """The ZIP route honours opts.initial_voltage (fpi.py:141-145) and raises the
    reference's ValueError on a length mismatch before any device work."""
    base = build_network(GenSpec(n_buses=9, seed=0))
    b = base.n_demand
    z = ZipCoefficients(alpha_z=np.full(b, 0.3), alpha_i=np.full(b, 0.3), alpha_p=np.full(b, 0.4))
    model = NetworkModel.from_branches(base.branches, 9, slack=base.slack, zip_coeffs=z)
    loads = LoadMatrix(np.full((b, 3), 0.01 + 0.005j))
    with pytest.raises(ValueError, match="initial voltage length mismatch"):
        batch_solve_dense(model, loads, SolveOptions(initial_voltage=np.ones(b + 1)))


@pytest.mark.parametrize("n_buses,seed", [(3, 0), (9, 1), (35, 0), (101, 2), (301, 3), (1001, 0), (5001, 0)])
def test_subtree_schedule_emulation_bitwise(n_buses, seed):
    """The warp-per-subtree schedule (positions, private top copies, Proot parity,
    child lists, Hu list-scheduled slots) solves Y_dd x = rhs with exactly the
    level kernel's operations: bit-identical to the level-order emulation."""
    from paper_2403_04578_b200 import sparse as sp
    from paper_2403_04578_b200._device import ModelContract, host_csr
    from paper_2403_04578_b200.subtree import subtree_schedule, subtree_solve_host, SUB_MAX_NS
    m = build_network(GenSpec(n_buses=n_buses, seed=seed))
    c = ModelContract.of(m)
    t = sp.tree_levels(sp.factorize_ydd(c.y_dd, count=False), c.src)
    s = subtree_schedule(t, *host_csr(c))
    if n_buses <= 3:  # a single level: no subtree below a top, the level kernel takes it
        assert s is None
        return
    assert s is not None and s.NS <= SUB_MAX_NS
    # every node appears once per copy: subtree nodes once, top nodes once per warp
    m_at = s.m_at[s.m_at >= 0]
    counts = np.bincount(m_at, minlength=c.b)
    top = counts > 1
    assert np.all(counts[~top] == 1) and np.all(counts[top] == s.W)
    rng = np.random.default_rng(seed)
    rhs = rng.standard_normal(c.b) + 1j * rng.standard_normal(c.b)
    assert np.array_equal(subtree_solve_host(s, rhs), sp.tree_solve_host(t, rhs))


@pytest.mark.parametrize("n_buses,seed", [(12, 1), (101, 0), (1001, 2)])
def test_tree_direct_solves_like_superlu(n_buses, seed):
    """The direct tree elimination (sparse.tree_direct, the radial feeders'
    batch factorization) solves Y_dd x = r like the SuperLU-based layout and
    dense LAPACK, with the same level structure."""
    from paper_2403_04578_b200 import GenSpec, build_network
    from paper_2403_04578_b200.sparse import ModelContract, factorize_ydd, tree_direct, tree_levels, tree_solve_host
    c = ModelContract.of(build_network(GenSpec(n_buses=n_buses, seed=seed)))
    td = tree_direct(c.y_dd, c.src)
    tl = tree_levels(factorize_ydd(c.y_dd, count=False), c.src)
    assert td is not None and td.levels == tl.levels
    assert np.array_equal(np.diff(td.level_info[:td.levels + 1]), np.diff(tl.level_info[:tl.levels + 1]))
    rng = np.random.default_rng(seed)
    r = rng.standard_normal(c.b) + 1j * rng.standard_normal(c.b)
    xe = np.linalg.solve(c.y_dd.toarray(), r)
    assert np.abs(tree_solve_host(td, r) - xe).max() <= 1e-12 * np.abs(xe).max()


def test_tree_direct_rejects_meshed_networks_and_counts_once():
    from paper_2403_04578_b200 import Branch, GenSpec, NetworkModel, build_network
    from paper_2403_04578_b200.sparse import ModelContract, factorization_count, radial_levels, tree_direct
    base = build_network(GenSpec(n_buses=40, seed=2))
    y0 = base.admittance.y_dd.toarray()
    i, j = next((i, j) for i in range(1, 40) for j in range(i + 2, 40) if y0[i - 1, j - 1] == 0)
    branches = list(base.branches) + [Branch(from_bus=i, to_bus=j, r=0.02, x=0.03)]  # a tie: one loop
    meshed = NetworkModel.from_branches(branches, 40, slack=base.slack)
    assert meshed.admittance.y_dd.nnz == base.admittance.y_dd.nnz + 2
    assert tree_direct(meshed.admittance.y_dd, meshed.source_injection()) is None
    c = ModelContract.of(base)
    n0 = factorization_count()
    assert radial_levels(c) is not None and factorization_count() == n0 + 1
    assert radial_levels(c, count=False) is not None and factorization_count() == n0 + 1
