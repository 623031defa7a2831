"""File layer at C2 size (525,600 cases x 100 nodes): native table reader/writer
vs the reference's Python loops (timed on a sample, extrapolated), and the CLI
solve end to end.  Writes under $TMPDIR."""
import json
import os
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, fileio, VoltageBatch  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 525600
d = tempfile.mkdtemp()
spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
L = gen_scenarios(m, tau, spec)
out = {"tau": tau, "b": 100, "host_threads": os.cpu_count()}
fileio.write_network(os.path.join(d, "net.json"), m)
t = time.perf_counter(); fileio.write_loads(os.path.join(d, "loads.csv"), L); out["native_write_loads_s"] = time.perf_counter() - t
out["loads_bytes"] = os.path.getsize(os.path.join(d, "loads.csv"))
t = time.perf_counter(); R = fileio.read_loads(os.path.join(d, "loads.csv")); out["native_read_loads_s"] = time.perf_counter() - t
assert np.array_equal(R.values, L.values)
vb = VoltageBatch(values=L.values * 0 + 1.0 - 0.01 * L.values, iterations=7, converged_mask=np.ones(tau, bool),
                  residuals=np.zeros(tau))
t = time.perf_counter(); fileio.write_voltages(os.path.join(d, "v.csv"), vb); out["native_write_voltages_s"] = time.perf_counter() - t
# reference-style Python loops on a sample, extrapolated
n = 5000
sub = fileio.LoadMatrix(values=L.values[:, :n])
t = time.perf_counter()
with open(os.path.join(d, "ref_loads.csv"), "w") as fh:
    fh.write(",".join(fileio._load_header(100)) + "\n")
    for j in range(n):
        cells = []
        for v in sub.values[:, j]:
            cells += [f"{v.real:.17g}", f"{v.imag:.17g}"]
        fh.write(",".join(cells) + "\n")
out["python_write_loads_s_extrapolated"] = (time.perf_counter() - t) * tau / n
t = time.perf_counter(); fileio._read_loads_python(os.path.join(d, "ref_loads.csv"))
out["python_read_loads_s_extrapolated"] = (time.perf_counter() - t) * tau / n
# CLI end to end on the GPU
t = time.perf_counter()
r = subprocess.run([sys.executable, "-m", "paper_2403_04578_b200", "solve", "--network", os.path.join(d, "net.json"),
                    "--loads", os.path.join(d, "loads.csv"), "--out", os.path.join(d, "vsolve.csv")],
                   capture_output=True, text=True)
out["cli_solve_wall_s"] = time.perf_counter() - t
out["cli_rc"] = r.returncode
meta = json.load(open(os.path.join(d, "vsolve.csv.meta.json")))
out["cli_solve_call_s"] = meta["wall_seconds"]
print(json.dumps(out))
