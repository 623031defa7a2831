"""Generate the file-format fixtures with the REFERENCE tpflow CLI (run in the
build container, where /root/reference exists; the outputs are committed).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_fileio.py

Writes tests/golden/fileio/: net9.json (gen-net), loads9.csv (gen-loads,
tau 50), heavy9.csv (one infeasible case: NaN voltages), and the reference
``solve`` outputs v9_{dense,sparse}.csv, heavy9_dense.csv (+ .meta.json).
"""
import os
import sys

from tpflow.cli import main

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fileio")
os.makedirs(OUT, exist_ok=True)


def run(*argv):
    rc = main([str(a) for a in argv])
    assert rc == 0, argv


def p(name):
    return os.path.join(OUT, name)


run("gen-net", "--buses", 9, "--seed", 0, "--out", p("net9.json"))
run("gen-loads", "--network", p("net9.json"), "--tau", 50, "--seed", 3, "--out", p("loads9.csv"))
with open(p("heavy9.csv"), "w") as fh:
    fh.write(",".join(f"p_{i},q_{i}" for i in range(1, 9)) + "\n")
    fh.write(",".join(["0.01,0.004"] * 8) + "\n")
    fh.write(",".join(["30.0,20.0"] * 8) + "\n")
for m in ("dense", "sparse"):
    run("solve", "--network", p("net9.json"), "--loads", p("loads9.csv"), "--method", m, "--out", p(f"v9_{m}.csv"))
run("solve", "--network", p("net9.json"), "--loads", p("heavy9.csv"), "--method", "dense", "--out",
    p("heavy9_dense.csv"))
# the reference solution the voltage files were written from (for writer byte tests)
import numpy as np  # noqa: E402
from tpflow import batch_solve_dense, fileio  # noqa: E402
from tpflow.fpi import SolveOptions  # noqa: E402
b = batch_solve_dense(fileio.read_network(p("net9.json")), fileio.read_loads(p("loads9.csv")), SolveOptions())
np.savez(p("v9_dense_batch.npz"), values=b.values, converged_mask=b.converged_mask)
print("wrote", sorted(os.listdir(OUT)), file=sys.stderr)
