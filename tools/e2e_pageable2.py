"""C2 through batch_solve_dense from a pageable array: with the K/W memo kept,
cleared per call (setup inside, as bench.py times it), and cleared with the
BLAS pool limited to one thread.  python tools/e2e_pageable2.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, LoadMatrix, batch_solve_dense  # noqa: E402
from paper_2403_04578_b200 import dense as dense_mod  # noqa: E402

spec = GenSpec(n_buses=101, seed=0)
m = build_network(spec)
loads = gen_scenarios(m, 525600, spec)
pinned = LoadMatrix(torch.from_numpy(loads.values).pin_memory().numpy())


def run(L, clear, n=4):
    o = batch_solve_dense(m, L)
    del o
    ts = []
    for _ in range(n):
        if clear:
            dense_mod._KW_CACHE.clear()
        t0 = time.perf_counter()
        o = batch_solve_dense(m, L)
        ts.append(time.perf_counter() - t0)
        del o
    return 1e3 * min(ts), 1e3 * sum(ts) / len(ts)


print("pinned   memo     min %.1f mean %.1f" % run(pinned, False))
print("pinned   cleared  min %.1f mean %.1f" % run(pinned, True))
print("pageable memo     min %.1f mean %.1f" % run(loads, False))
print("pageable cleared  min %.1f mean %.1f" % run(loads, True))
from threadpoolctl import threadpool_limits  # noqa: E402
with threadpool_limits(limits=1, user_api="blas"):
    print("pageable cleared, BLAS 1 thread  min %.1f mean %.1f" % run(loads, True))

# the inverse with the library's threads (bitwise the reference's K), then the
# pool limited to one thread for the copies: do the spinning workers park?
orig = dense_mod.dense_kw


def kw_then_park(c):
    r = orig(c)
    threadpool_limits(limits=1, user_api="blas")  # not restored: measure the effect
    return r


dense_mod.dense_kw = kw_then_park
print("pageable cleared, park after inverse  min %.1f mean %.1f" % run(loads, True))
