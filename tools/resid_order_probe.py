"""C2 residual with the rows in index order vs a depth-first order of the
feeder (tpf_residual_order_c128): time and bits.  python tools/resid_order_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy.sparse import csgraph  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator, _capi  # noqa: E402
from paper_2403_04578_b200._device import complex_strides, stream_ptr  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
op = DenseOperator(m, "cuda:0")
S = gen_scenarios_device(m, 525600, spec, device="cuda:0")
V, it = op.solve(S)
rp, ci, yv, src, _ = op.contract.csr_on(op.device)
y = m.admittance.y_dd.tocsr()
roots = np.nonzero(op.contract.src != 0)[0]
order = np.concatenate([csgraph.depth_first_order(abs(y), int(r), directed=False, return_predecessors=False)
                        for r in roots])
order = np.concatenate([order, np.setdiff1d(np.arange(op.b), order)]).astype(np.int32)
dorder = torch.from_numpy(order).cuda()
r1 = torch.empty(525600, dtype=torch.float64, device="cuda:0")
r2 = torch.empty_like(r1)
sn, sc = complex_strides(S)
vn, vc = complex_strides(V)


def run(out, ordp):
    _capi.call("tpf_residual_order_c128", 525600, op.b, S.data_ptr(), sn, sc, V.data_ptr(), vn, vc, rp.data_ptr(),
               ci.data_ptr(), yv.data_ptr(), src.data_ptr(), ordp, out.data_ptr(), stream_ptr(op.device))


for name, out, ordp in (("index order", r1, 0), ("depth-first", r2, dorder.data_ptr())):
    run(out, ordp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run(out, ordp)
    e1.record()
    torch.cuda.synchronize()
    print("%-12s %.3f ms" % (name, e0.elapsed_time(e1) / 10))
print("same bits:", bool(torch.equal(r1, r2)))
