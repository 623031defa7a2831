"""C2 end to end from pinned host memory, split: setup (K, W) alone, the
whole public call, and chunk-size / ramp variants of the host pipeline.
python tools/c2_e2e_split.py"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense  # noqa: E402
from paper_2403_04578_b200 import dense as dense_mod  # noqa: E402
from paper_2403_04578_b200._device import ModelContract  # noqa: E402


def tm(f, n=5, clear=True):
    f()
    ts = []
    for _ in range(n):
        if clear:
            dense_mod._KW_CACHE.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del r
    return 1e3 * min(ts), 1e3 * sum(ts) / len(ts)


spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
if len(sys.argv) > 1:  # child: one pipeline setting from the environment
    loads = gen_scenarios(m, 525600, spec)
    host = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())
    ch = int(os.environ.get("CHUNK", "0"))
    print(sys.argv[1], "call min %.2f mean %.2f ms" % tm(lambda: batch_solve_dense(m, host, chunk_cases=ch)))
    sys.exit(0)
c = ModelContract.of(m)
dev = torch.device("cuda", 0)
print("setup operator_kw (device) min %.3f mean %.3f ms" % tm(lambda: dense_mod.operator_kw(c, dev)))
for name, env in (("default", {}), ("ramp/8", {"TPF_PIPE_RAMP_DIV": "8"}), ("ramp/16", {"TPF_PIPE_RAMP_DIV": "16"}),
                  ("chunk 16384", {"CHUNK": "16384"}), ("chunk 24576", {"CHUNK": "24576"}),
                  ("chunk 49152", {"CHUNK": "49152"}), ("chunk 65536", {"CHUNK": "65536"})):
    out = subprocess.run([sys.executable, __file__, name], env=dict(os.environ, **env), capture_output=True,
                         text=True)
    print(out.stdout.strip() or out.stderr[-300:])
