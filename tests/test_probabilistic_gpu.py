"""Probabilistic power flow (config C4, probabilistic.probabilistic_pf): scenario
batches generated, solved and reduced on the device; the statistics against a
direct solve of the same batches, and sampled columns against the CPU oracle
(SURVEY 7 "Config 4": sub-batches verified against the oracle)."""

import numpy as np
import pytest

from conftest import gpu_available
from oracle import tpf_oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("method", ["dense", "sparse"])
def test_probabilistic_pf_stats_and_sampled_parity(method):
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator, SparseOperator, SolveOptions
    from paper_2403_04578_b200.probabilistic import probabilistic_pf
    from paper_2403_04578_b200.synth import gen_scenarios_device
    n_buses = 101 if method == "dense" else 301
    model = build_network(GenSpec(n_buses=n_buses, seed=0))
    tau, n_scen = 70_000, 3
    rng = np.random.default_rng(7)
    sample = {s: np.sort(rng.choice(tau, 40, replace=False)) for s in (0, 2)}
    st = probabilistic_pf(model, n_scen, tau, method=method, sample=sample)
    # the same batches solved directly (same generator seeds -> same loads)
    op = DenseOperator(model) if method == "dense" else SparseOperator(model)
    mags, its = [], []
    for s in range(n_scen):
        S = gen_scenarios_device(model, tau, GenSpec(n_buses=n_buses, seed=1000 + s), device="cuda:0")
        V, it = op.solve(S, SolveOptions())
        mags.append(V.abs())
        its.append(it)
    A = torch.cat(mags, dim=1)
    # |V| as hypot in the kernel; torch's complex abs may differ in the last bit
    assert np.allclose(st.vmin, A.min(dim=1).values.cpu().numpy(), rtol=5e-16, atol=0)
    assert np.allclose(st.vmax, A.max(dim=1).values.cpu().numpy(), rtol=5e-16, atol=0)
    assert np.allclose(st.vmean, A.mean(dim=1).cpu().numpy(), rtol=1e-13, atol=0)
    assert st.sum_iterations == int(sum(int(i.sum()) for i in its))
    assert st.max_iterations == max(int(i.max()) for i in its)
    assert st.nonconverged == 0 and st.n_cases == n_scen * tau
    y, src, v_s = model.admittance.y_dd, model.source_injection(), model.slack.v_s
    for s, (cols, Ss, Vs, it_s) in st.samples.items():
        Vo, n, mask, _ = orc.dense_per_case(y, src, v_s, Ss)
        assert mask.all()
        assert np.abs(Vs - Vo).max() < 1e-12
        assert np.abs(it_s.astype(int) - n).max() <= 1
