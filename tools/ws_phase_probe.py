"""Per-role cycle accounting of the warp-specialised dense kernel (debug build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator, _capi
lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "build_timing", "libtpf_timing.so"))
for name, (res, args) in _capi.SIGNATURES.items():
    fn = getattr(lib, name, None)
    if fn is not None:
        fn.restype, fn.argtypes = res, args
spec = GenSpec(n_buses=101, seed=0); model = build_network(spec)
tau = 525600
S = torch.from_numpy(gen_scenarios(model, tau, spec).values).cuda()
op = DenseOperator(model)
V = torch.empty_like(S); it = torch.empty(tau, dtype=torch.int32, device="cuda")
ws = torch.empty(256, dtype=torch.uint8, device="cuda")
def run():
    assert lib.tpf_dense_ws_fpi_c128(tau, 100, S.data_ptr(), tau, 1, op.K.data_ptr(), op.W.data_ptr(), 1.0, 0.0,
                                     1e-10, 100, V.data_ptr(), tau, 1, it.data_ptr(), ws.data_ptr(), 256,
                                     torch.cuda.current_stream().cuda_stream) == 0
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
print("kernel ms (timing build)", e0.elapsed_time(e1), "sum_n", int(it.sum()))
buf = np.zeros((148 * 12, 8), dtype=np.int64)
lib.tpf_debug_ws_phase_cycles(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
b = buf.reshape(148, 12, 8)
mma = b[:, 0:4].reshape(-1, 8); ew = b[:, 4:12].reshape(-1, 8)
print("MMA: rounds %.0f, wait-U %.1f%%, gemm %.1f%%, per-round gemm %.0f clk wait %.0f clk, DMMA/round %d" % (
    mma[:, 6].mean(), 100 * mma[:, 0].mean() / mma[:, 7].mean(), 100 * mma[:, 1].mean() / mma[:, 7].mean(),
    mma[:, 1].mean() / mma[:, 6].mean(), mma[:, 0].mean() / mma[:, 6].mean(), 13 * 25 * 3))
print("EW GEMM share: %.0f clk per round (%.1f%%)" % (ew[:, 1].mean() / ew[:, 6].mean(), 100 * ew[:, 1].mean() / ew[:, 7].mean()))
names = ["U round", "wait V'", "test", "retire/refill"]
print("EW: rounds %.0f" % ew[:, 6].mean(), " ".join("%s %.0f clk (%.1f%%)" % (n, ew[:, 2 + i].mean() / ew[:, 6].mean(),
      100 * ew[:, 2 + i].mean() / ew[:, 7].mean()) for i, n in enumerate(names)))
