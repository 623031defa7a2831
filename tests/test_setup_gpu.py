"""Dense setup on the device (A3, dense.py:150-152): K = -inv(Y_dd) and W = K src
from tree-LU solves (tpf_dense_setup_tree_c128) against the reference's LAPACK
inverse, and the solves that use them."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _model(nb, seed=0, load_scale=1.0):
    from paper_2403_04578_b200 import GenSpec, build_network
    return build_network(GenSpec(n_buses=nb, seed=seed, load_scale=load_scale))


@pytest.mark.parametrize("nb", [12, 101, 301, 1001])
def test_device_kw_matches_lapack(nb):
    import torch
    from paper_2403_04578_b200._device import ModelContract
    from paper_2403_04578_b200.dense import dense_kw, device_kw
    c = ModelContract.of(_model(nb, seed=nb))
    Kh, Wh = dense_kw(c)
    kw = device_kw(c, torch.device("cuda", 0))
    assert kw is not None
    Kd, Wd = (x.cpu().numpy() for x in kw)
    assert np.abs(Kd - Kh).max() <= 1e-13 * np.abs(Kh).max()
    assert np.abs(Wd - Wh).max() <= 1e-13 * np.abs(Wh).max()
    # a second call is the memoised pair, the same tensors
    kw2 = device_kw(c, torch.device("cuda", 0))
    assert kw2[0] is kw[0]


def test_meshed_network_keeps_host_setup(golden):
    from paper_2403_04578_b200 import DenseOperator
    g = golden("asym6")
    op = DenseOperator(g.model, setup="device")
    assert op.setup == "host"  # no zero-fill tree elimination: LAPACK, as the reference


def test_auto_setup_choice():
    from paper_2403_04578_b200 import DenseOperator
    assert DenseOperator(_model(101)).setup == "device"          # radial feeders: on the device
    assert DenseOperator(_model(35)).setup == "host"             # small: LAPACK is cheaper
    assert DenseOperator(_model(101), setup="host").setup == "host"  # LAPACK, bitwise the reference's K
    with pytest.raises(ValueError):
        DenseOperator(_model(101), setup="gpu")


def test_c5_golden_with_device_setup(golden):
    """Near voltage collapse (C5, b = 1,000): the device K gives the reference's
    batch count and mask and its voltages to the golden tolerance."""
    import torch
    from paper_2403_04578_b200 import DenseOperator
    g = golden("c5_slice32")
    ops = {s: DenseOperator(g.model, setup=s) for s in ("host", "device")}
    assert ops["device"].setup == "device"
    S = torch.from_numpy(g.S).cuda()
    (Vh, ih), (Vd, idv) = (ops[s].solve(S, g.opts()) for s in ("host", "device"))
    assert int(idv.max()) == int(g["dense_iterations"]) == 58
    assert (Vd - Vh).abs().max().item() <= 1e-11
    assert (idv - ih).abs().max().item() <= 1
    assert np.abs(Vd.cpu().numpy() - g["dense_V"]).max() <= 1e-9


def test_host_pipeline_with_device_setup_matches_device_path():
    """batch_solve_dense (host buffers, K and W from the device setup at b >= 256)
    equals the device-resident operator bitwise."""
    import torch
    from paper_2403_04578_b200 import DenseOperator, batch_solve_dense, gen_scenarios, GenSpec
    m = _model(301, seed=3)
    loads = gen_scenarios(m, 700, GenSpec(n_buses=301, seed=3))
    out = batch_solve_dense(m, loads)
    op = DenseOperator(m)
    assert op.setup == "device"
    V, it = op.solve(torch.from_numpy(np.ascontiguousarray(loads.values)).cuda())
    assert np.array_equal(out.values, V.cpu().numpy())
    assert np.array_equal(out.iterations_per_case, it.cpu().numpy())
