"""Per-phase cycle accounting of the dense kernel (debug build, tools/build_timing.sh)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator
from paper_2403_04578_b200 import _capi

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "build_timing", "libtpf_timing.so"))
for name, (res, args) in _capi.SIGNATURES.items():
    fn = getattr(lib, name, None)
    if fn is not None:
        fn.restype, fn.argtypes = res, args
spec = GenSpec(n_buses=101, seed=0)
model = build_network(spec)
tau = int(sys.argv[1]) if len(sys.argv) > 1 else 525600
S = torch.from_numpy(gen_scenarios(model, tau, spec).values).cuda()
op = DenseOperator(model)
V = torch.empty_like(S); it = torch.empty(tau, dtype=torch.int32, device="cuda")
ws = torch.empty(256, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def run():
    rc = lib.tpf_dense_fpi_c128(tau, 100, S.data_ptr(), tau, 1, op.K.data_ptr(), op.W.data_ptr(), 1.0, 0.0, 1e-10, 100,
                                V.data_ptr(), tau, 1, it.data_ptr(), ws.data_ptr(), 256, st)
    assert rc == 0, lib.tpf_last_error()
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
print("kernel ms (timing build)", e0.elapsed_time(e1))
buf = np.zeros((148 * 16, 8), dtype=np.int64)
lib.tpf_debug_phase_cycles(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), 148 * 16)
w = buf[:148 * 8]
names = ["elementwise", "bar_U", "gemm", "epilogue", "bar_flags", "retire/refill"]
tot = w[:, 7].astype(float)
print("iterations per warp mean", w[:, 6].mean(), "cycles total mean %.3e" % tot.mean())
for i, n in enumerate(names):
    print(f"{n:14s} {w[:, i].mean() / tot.mean():6.1%}  per-iter {w[:, i].mean() / w[:, 6].mean():8.0f} clk")
# by warp role (half 0 / half 1, big/small)
for h in range(8):
    sel = w[h::8]
    print("warp", h, " ".join(f"{sel[:, i].mean() / sel[:, 6].mean():7.0f}" for i in range(6)))
