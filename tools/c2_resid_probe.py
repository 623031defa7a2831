"""Standalone residual kernel at C2 (b=100, tau=525,600) for row-block counts
given in TPF_RESID_NRB: time and bitwise agreement.  python tools/c2_resid_probe.py
(measured: 0.49-0.52 ms for every count, the same bits; a shared-memory tile
variant staging 32 cases' V columns ran 1.03 ms and was dropped)"""
import os
import subprocess
import sys

if len(sys.argv) > 1:  # child: one setting
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, DenseOperator
    from paper_2403_04578_b200._device import residual_and_summary
    from paper_2403_04578_b200.synth import gen_scenarios_device
    spec = GenSpec(n_buses=101, seed=0)
    m = build_network(spec)
    op = DenseOperator(m, "cuda:0")
    S = gen_scenarios_device(m, 525600, spec, device="cuda:0")
    V, it = op.solve(S)
    csr = op.contract.csr_on(op.device)
    out = (torch.empty(525600, dtype=torch.float64, device="cuda:0"),
           torch.empty(525600, dtype=torch.uint8, device="cuda:0"), torch.empty(2, dtype=torch.int32, device="cuda:0"))
    f = lambda: residual_and_summary(op.contract, S, V, it, 1e-8, op.device, csr=csr, out=out)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    np.save(sys.argv[1], out[0].cpu().numpy())
    print(os.environ.get("TPF_RESID_NRB", "auto"), "%.3f ms" % (e0.elapsed_time(e1) / 10))
else:
    res = {}
    for nrb in ("1", "2", "3", "4", "6"):
        env = dict(os.environ, TPF_RESID_NRB=nrb)
        path = f"/tmp/resid_{nrb}.npy"
        print(subprocess.run([sys.executable, __file__, path], env=env, capture_output=True, text=True).stdout.strip())
        import numpy as np
        res[nrb] = np.load(path)
    print("bitwise equal to nrb=1:", {k: bool(np.array_equal(v.view(np.uint64), res["1"].view(np.uint64))) for k, v in res.items()})
