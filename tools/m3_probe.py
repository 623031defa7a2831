"""3M vs 4M GEMM in the ws kernel: counts and values at full C2 (numpy loads)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator  # noqa: E402

if len(sys.argv) > 1:  # child: solve with the env's kernel choice, save
    spec = GenSpec(n_buses=101, seed=0)
    model = build_network(spec)
    S = torch.from_numpy(gen_scenarios(model, 525600, spec).values).cuda()
    V, it = DenseOperator(model).solve(S, kernel="ws")
    np.savez(sys.argv[1], V=V.cpu().numpy(), it=it.cpu().numpy())
    sys.exit(0)
env = dict(os.environ)
subprocess.check_call([sys.executable, __file__, "/tmp/m3.npz"], env=env)
env["TPF_WS_4M"] = "1"
subprocess.check_call([sys.executable, __file__, "/tmp/m4.npz"], env=env)
a, b = np.load("/tmp/m3.npz"), np.load("/tmp/m4.npz")
d = a["it"].astype(int) - b["it"].astype(int)
print("sum n 3M", a["it"].sum(), "4M", b["it"].sum(), "cases differing", int((d != 0).sum()), "max |dn|", int(abs(d).max()))
same = d == 0
print("max |dV| (same counts)", float(np.abs(a["V"][:, same] - b["V"][:, same]).max()))
print("max |dV| (all)", float(np.abs(a["V"] - b["V"]).max()))
