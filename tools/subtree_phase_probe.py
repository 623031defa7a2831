"""Per-phase cycle accounting of the warp-per-subtree sparse kernel (debug build:
TPF_EXTRA_DEFS= tools/build_timing.sh).  python tools/subtree_phase_probe.py [tau] [case|node]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, _capi  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "build_timing", "libtpf_timing.so"))
for name, (res, args) in _capi.SIGNATURES.items():
    fn = getattr(lib, name, None)
    if fn is not None:
        fn.restype, fn.argtypes = res, args
_capi._lib = lib  # route the operator through the debug build
tau = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
spec = GenSpec(n_buses=5001, seed=0)
m = build_network(spec)
op = SparseOperator(m, "cuda:0")
S = gen_scenarios_device(m, tau, spec, device="cuda:0")
if len(sys.argv) > 2 and sys.argv[2] == "case":
    S = S.t().contiguous().t()
r = torch.empty(tau, dtype=torch.float64, device="cuda:0")
V, it = op.solve(S, resid=r, V=torch.empty_like(S))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
V, it = op.solve(S, V=V, iters=it, resid=r)
e1.record()
torch.cuda.synchronize()
print("ms (timing build)", e0.elapsed_time(e1), "kernel", op.kernel)
buf = np.zeros(148 * 12, dtype=np.int64)
lib.tpf_debug_subtree_phase_cycles(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
b = buf.reshape(148, 12).astype(float)
cases, iters = b[:, 8].sum(), b[:, 9].sum()
names = ["load", "subtree up", "barrier wait", "top", "subtree down", "retire+store", "residual", "end barrier"]
tot = b[:, 10].sum()
print("cases %.0f iterations %.0f (%.2f per case); cycles per case %.0f" % (cases, iters, iters / cases, tot / cases))
for i, n in enumerate(names):
    per_it = i in (1, 2, 3, 4)
    print("%-14s %5.1f%%  %8.0f cycles per %s" % (n, 100 * b[:, i].sum() / tot, b[:, i].sum() / (iters if per_it else cases),
                                             "iteration" if per_it else "case"))
