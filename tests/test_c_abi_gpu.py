"""The C boundary from C: tests/c_abi/solve_host.c is compiled with gcc
against include/tpf.h and libtpf.so and solves a batch from host buffers;
its voltages and counts equal the Python API's bit for bit."""

import os
import shutil
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_caller_matches_python(tmp_path):
    from paper_2403_04578_b200 import GenSpec, LoadMatrix, batch_solve_dense, build_network, gen_scenarios
    from paper_2403_04578_b200._device import ModelContract, host_csr
    from paper_2403_04578_b200.dense import dense_kw
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    pkg = os.path.join(ROOT, "paper_2403_04578_b200")
    exe = str(tmp_path / "solve_host")
    cuda_lib = "/usr/local/cuda/lib64"
    subprocess.run([cc, "-O2", "-o", exe, os.path.join(ROOT, "tests", "c_abi", "solve_host.c"),
                    "-I", os.path.join(ROOT, "include"), "-L", pkg, "-ltpf", "-L", cuda_lib, "-lcudart",
                    f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{cuda_lib}"], check=True)
    spec = GenSpec(n_buses=35, seed=7)
    m = build_network(spec)
    loads = gen_scenarios(m, 3000, spec)
    c = ModelContract.of(m)
    K, W = dense_kw(c)  # the host LAPACK setup at b = 34 (what batch_solve_dense uses there)
    rp, ci, yv = host_csr(c)
    ind, outd = tmp_path / "in", tmp_path / "out"
    ind.mkdir()
    outd.mkdir()
    for name, arr in (("dims", np.array([c.b, 3000], np.int64)), ("K", K), ("W", W), ("rp", rp), ("ci", ci),
                      ("yv", yv), ("src", c.src), ("S", np.ascontiguousarray(loads.values)),
                      ("vflat", np.array([abs(c.v_s), 0.0]))):
        np.ascontiguousarray(arr).tofile(str(ind / f"{name}.bin"))
    r = subprocess.run([exe, str(ind), str(outd)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    it_max, n_conv = (int(x) for x in r.stdout.split())
    V = np.fromfile(str(outd / "V.bin"), dtype=np.complex128).reshape(c.b, 3000)
    it = np.fromfile(str(outd / "iters.bin"), dtype=np.int32)
    ref = batch_solve_dense(m, LoadMatrix(loads.values))
    assert np.array_equal(V, ref.values)
    assert np.array_equal(it, ref.iterations_per_case)
    assert it_max == ref.iterations and n_conv == int(ref.converged_mask.sum())
