#!/bin/bash
# A/B of the dense ws kernel prologue: K^T image by cp.async.bulk (default) vs per-CTA gather
cd "$(dirname "$0")/.."
for g in 0 1 2 0 1 2; do
  TPF_WS_GATHER=$g python - <<'PY'
import os, torch
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator
spec = GenSpec(n_buses=101, seed=0); model = build_network(spec)
S = torch.from_numpy(gen_scenarios(model, 525600, spec).values).cuda()
op = DenseOperator(model); V = torch.empty_like(S); it = torch.empty(525600, dtype=torch.int32, device="cuda")
for _ in range(3): op.solve(S, V=V, iters=it, kernel="ws")
torch.cuda.synchronize(); ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); op.solve(S, V=V, iters=it, kernel="ws"); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("TPF_WS_GATHER=%s min %.3f med %.3f" % (os.environ["TPF_WS_GATHER"], min(ts), sorted(ts)[5]), int(it.sum()))
PY
done
