"""Per-phase cycle accounting of the sparse tree kernel (debug build, tools/build_timing.sh)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, _capi  # noqa: E402
from paper_2403_04578_b200.synth import gen_scenarios_device  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", os.environ.get("TPF_TIMING_DIR", "build_timing"), "libtpf_timing.so"))
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
r = torch.empty(tau, dtype=torch.float64, device="cuda:0")
V, it = op.solve(S, resid=r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
V, it = op.solve(S, V=V, iters=it, resid=r)
e1.record()
torch.cuda.synchronize()
print("kernel ms (timing build)", e0.elapsed_time(e1), "levels", op.tree.levels, "slots", op.tree.slots)
buf = np.zeros(148 * 8, dtype=np.int64)
lib.tpf_debug_tree_phase_cycles(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
b = buf.reshape(148, 8).astype(float)
cases, iters = b[:, 5].sum(), b[:, 6].sum()
names = ["load", "up-sweep", "down-sweep", "retire", "residual"]
tot = b[:, 7].mean()
print("cases %.0f iterations %.0f (%.2f per case)" % (cases, iters, iters / cases))
for i, n in enumerate(names):
    per = b[:, i].sum() / (iters if i in (1, 2) else cases)
    print("%-10s %5.1f%% of time, %8.0f clk per %s" % (n, 100 * b[:, i].mean() / tot, per,
                                                       "iteration" if i in (1, 2) else "case"))
