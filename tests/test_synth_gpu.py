"""Device scenario generator (synth.gen_scenarios_device) against the
reference model it restates (synth.py:131-156): not bit-identical (Philox on the
device vs PCG64 in numpy), so the test checks the model's statistics and its
deterministic parts exactly."""

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _stats(S, base):
    p, q = S.real, S.imag
    pf = p / np.abs(S)
    lp = np.log(p)
    lat = lp - lp.mean(axis=1, keepdims=True)
    corr = np.corrcoef(lat[:8])[np.triu_indices(8, 1)]
    return dict(pf_min=pf.min(), pf_max=pf.max(), pf_mean=pf.mean(), pf_std=pf.std(),
                q_min=q.min(), sigma=lat.std(axis=1), corr=corr,
                base_ratio=np.exp(lp.mean(axis=1) - lp.mean(axis=1)[0]) / (base / base[0]))


def test_gen_scenarios_device_statistics_and_scaling():
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios
    from paper_2403_04578_b200.synth import gen_scenarios_device, scenario_margin
    spec = GenSpec(n_buses=101, seed=0, load_scale=1.0)
    model = build_network(spec)
    tau = 200_000
    Sd = gen_scenarios_device(model, tau, spec, device="cuda:0", chunk=1 << 15).cpu().numpy()
    Sh = gen_scenarios(model, 50_000, spec).values
    base = spec.stream(2).uniform(0.5, 1.5, size=model.n_demand)  # the same numpy draw both use
    # global scaling (synth.py:153-155): the worst aggregate sits exactly at load_scale x margin
    target = spec.load_scale * scenario_margin(model)
    assert np.abs(Sd.sum(axis=0)).max() == pytest.approx(target, rel=1e-12)
    assert np.abs(Sh.sum(axis=0)).max() == pytest.approx(target, rel=1e-12)
    d, h = _stats(Sd, base), _stats(Sh, base)
    for st in (d, h):
        assert 0.9 - 1e-12 <= st["pf_min"] and st["pf_max"] <= 1.0 + 1e-12  # U[0.9, 1] lagging
        assert st["q_min"] >= 0.0
        assert st["pf_mean"] == pytest.approx(0.95, abs=2e-3)
        assert st["pf_std"] == pytest.approx(0.1 / np.sqrt(12), abs=2e-3)
        assert np.all(np.abs(st["sigma"] - 0.4) < 0.02)        # lognormal sigma 0.4
        assert np.all(np.abs(st["corr"] - 0.5) < 0.04)          # one-factor correlation 0.5
        assert np.all(np.abs(st["base_ratio"] - 1.0) < 0.03)    # per-node base sizes
    # chunk independence: the same seed and chunking give the same batch
    Sd2 = gen_scenarios_device(model, tau, spec, device="cuda:0", chunk=1 << 15).cpu().numpy()
    assert np.array_equal(Sd, Sd2)
