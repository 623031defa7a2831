"""Per-scenario cost of the C4 pass (b=100, tau=525,600): generator, solve,
residual + summary, statistics.  python tools/c4_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator, SolveOptions, _capi  # noqa: E402
from paper_2403_04578_b200._device import residual_and_summary, complex_strides, stream_ptr  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device, scenario_margin  # noqa: E402

tau = 525600
model = build_network(GenSpec(n_buses=101, seed=0))
dev = torch.device("cuda", 0)
op = DenseOperator(model, dev)
b = op.b


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - w0) * 1e3 / n


spec = GenSpec(n_buses=101, seed=1000)
S = gen_scenarios_device(model, tau, spec, device=dev)
V = torch.empty_like(S)
it = torch.empty(tau, dtype=torch.int32, device=dev)
csr = op.contract.csr_on(dev)
post = (torch.empty(tau, dtype=torch.float64, device=dev), torch.empty(tau, dtype=torch.uint8, device=dev),
        torch.empty(2, dtype=torch.int32, device=dev))
lib = _capi.load()
vmin = torch.zeros(b, dtype=torch.float64, device=dev)
vmax, vsum = torch.zeros_like(vmin), torch.zeros_like(vmin)
ws = torch.empty(int(lib.tpf_voltage_stats_workspace_bytes(tau, b)), dtype=torch.uint8, device=dev)
vn, vc = complex_strides(V)
print("scenario_margin (host) ms/call: %.3f" % timed(lambda: scenario_margin(model))[1])
print("generator        ms (device, wall): %.3f %.3f" % timed(lambda: gen_scenarios_device(model, tau, spec, device=dev)))
print("solve            ms: %.3f %.3f" % timed(lambda: op.solve(S, SolveOptions(), V=V, iters=it)))
print("residual+summary ms: %.3f %.3f" % timed(lambda: residual_and_summary(op.contract, S, V, it, 1e-8, dev, csr=csr,
                                                                            out=post)))
print("voltage stats    ms: %.3f %.3f" % timed(lambda: _capi.call(
    "tpf_voltage_stats_c128", tau, b, V.data_ptr(), vn, vc, vmin.data_ptr(), vmax.data_ptr(), vsum.data_ptr(), 1,
    ws.data_ptr(), ws.numel(), stream_ptr(dev))))
