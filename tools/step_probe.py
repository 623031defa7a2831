"""Where does a bench step's time go?  GPU events vs CPU enqueue time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator
from paper_2403_04578_b200._device import residual_and_summary
spec = GenSpec(n_buses=101, seed=0); model = build_network(spec)
S = torch.from_numpy(gen_scenarios(model, 525600, spec).values).cuda()
op = DenseOperator(model); dev = S.device
V = torch.empty_like(S); it = torch.empty(525600, dtype=torch.int32, device=dev)
csr = op.contract.csr_on(dev)
post = (torch.empty(525600, dtype=torch.float64, device=dev), torch.empty(525600, dtype=torch.uint8, device=dev),
        torch.empty(2, dtype=torch.int32, device=dev))
def step(mode):
    op.solve(S, V=V, iters=it)
    if mode >= 1:
        residual_and_summary(op.contract, S, V, it, 1e-8, dev, csr=csr, out=post)
for mode in (0, 1, 0, 1):
    for _ in range(3): step(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = time.perf_counter(); e0.record()
    for _ in range(10): step(mode)
    c1 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); c2 = time.perf_counter()
    print(f"mode {mode}: gpu {e0.elapsed_time(e1)/10:.3f} ms/step, cpu enqueue {(c1-c0)*100:.3f} ms/step, wall {(c2-c0)*100:.3f}")
