"""Benchmark: power flows / s of the dense (default) or sparse TPF hot path.

Default workload = BASELINE.json configs[1] (C2): 100-node synthetic radial
feeder (GenSpec(101, seed=0)), tau = 525,600 one-minute steps, complex128,
FP64 tensor-core dense TPF on one B200.  Under torchrun each rank solves its own
525,600-case scenario batch (weak scaling, no data-path collective; rank r>0
uses scenario seed 1000+r); the job value is the sum of
cases over all ranks / the max-over-ranks device time.

Legs of one run (one JSON line on rank 0):
  value    device-resident: S already in HBM; per step = iteration kernel +
           residual post-check + summary (CUDA events, max over ranks);
  roofline dominant kernel (dense_fpi_kernel) vs the FP64 DMMA peak measured
           in-run by tpf_probe_fp64_tflops (MEASURED_PEAKS.json has no FP64);
  e2e      the public API batch_solve_dense(model, LoadMatrix(S_host)) from
           pinned host memory, H2D/D2H inside the timed region;
  cpu_baseline  oracle port of the reference batch_solve_dense (numpy, BLAS
           threads 1, workers = host cores) on a bounded sample (rank 0, N=1).
`--impl reference` times only the CPU reference port (rank 0), same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "power flows/sec (τ×scenarios solved) dense+sparse TPF at 1/2/4/8 B200 vs CPU"
UNIT = "power_flows/s"

CONFIGS = {
    # name: (n_buses, load seed (rank 0), tau, load_scale, method, description)
    "c2": (101, 0, 525600, 1.0, "dense", "C2 dense TPF, b=100, tau=525,600 (1-min year), complex128 DMMA"),
    "c1": (35, 0, 8760, 1.0, "dense", "C1 dense TPF, b=34, tau=8,760 (hourly year)"),
    "c5": (1001, 0, 8760, 21.0, "dense", "C5 dense TPF, b=1,000, load_scale 21 (near collapse), tau=8,760"),
    "c3": (5001, 0, 525600, 1.0, "sparse", "C3 sparse TPF, b=5,000, tau=525,600, batched LU trisolves"),
    "c4": (101, 1000, 525600, 1.0, "dense",
           "C4 probabilistic PF: 100-node feeder x 525,600 steps per scenario, one scenario batch per step "
           "(device-generated, scenario seed 1000+s), scenarios dealt round-robin over ranks"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    p.add_argument("--dtype", choices=["c128", "c64"], default="c128",
                   help="c64: the complex64 twin (FP32 SIMT, tol 1e-6), reported as its own line")
    p.add_argument("--tau", type=int, default=None, help="override tau (testing only)")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU sample duration")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--chunk-cases", type=int, default=0, help="e2e host-pipeline chunk (0 = library default)")
    p.add_argument("--no-graph", dest="graph", action="store_false",
                   help="time eager launches instead of a CUDA-graph replay of the step")
    p.add_argument("--scenarios", type=int, default=1000, help="c4: scenario batches in the timed pass")
    p.add_argument("--no-sparse", dest="sparse_half", action="store_false",
                   help="default (c2) line without the nested C3 sparse object")
    return p.parse_args()


ARGS = parse()
if ARGS.impl == "reference":
    # the reference's best CPU setting: BLAS single-threaded, workers = cores
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


HOST_GEN_LIMIT = 8 << 30  # bytes of S above which the value leg generates loads on the device


def workload(cfg, rank, host_tau=None):
    """(model, host LoadMatrix of host_tau cases or the full tau, method, description, tau, lspec)."""
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios
    n_buses, seed, tau, scale, method, desc = CONFIGS[cfg]
    if ARGS.tau:
        tau = ARGS.tau
    spec = GenSpec(n_buses=n_buses, seed=0, load_scale=scale)
    model = build_network(spec)
    lseed = seed if rank == 0 else 1000 + rank
    lspec = GenSpec(n_buses=n_buses, seed=lseed, load_scale=scale)
    loads = gen_scenarios(model, min(tau, host_tau) if host_tau else tau, lspec)
    return model, loads, method, desc, tau, lspec


def cpu_sample(model, loads, seconds, cores):
    """Time the oracle port of batch_solve_dense/sparse on a bounded column sample."""
    from threadpoolctl import threadpool_limits
    from oracle import tpf_oracle as orc
    y, src, v_s = model.admittance.y_dd, model.source_injection(), model.slack.v_s
    S = loads.values
    method = CONFIGS[ARGS.config][4]
    K, W = orc.dense_operators(y, src) if method == "dense" else (None, None)

    def run(cols):
        sub = np.ascontiguousarray(S[:, :cols])
        t0 = time.perf_counter()
        if method == "dense":
            with threadpool_limits(limits=1, user_api="blas"):
                orc.dense_joint(y, src, v_s, sub, workers=cores, K=K, W=W)
        else:
            orc.sparse_block(y, src, v_s, sub)
        return time.perf_counter() - t0

    cols = min(S.shape[1], 1024 if method == "dense" else 64)
    dt = run(cols)
    target = int(cols * seconds / max(dt, 1e-6) / 3)
    if method == "sparse":
        target = min(target, 1200)  # the reference's SuperLU fails from tau ~1,800
    cols = max(cols, min(S.shape[1], target))
    times = [run(cols) for _ in range(3)]
    t = float(np.median(times))
    out = dict(value=cols / t, unit=UNIT, cores=cores, kind="port", cpu=cpu_model(),
               sample=f"first {cols} of {S.shape[1]} cases, oracle port of tpflow.batch_solve_"
                      f"{method}, median of 3, setup (inverse) excluded, BLAS threads 1, "
                      f"workers={cores if method == 'dense' else 1}")
    if method == "dense":
        # BASELINE.md 3.3 secondary setting: the reference's defaults (workers=1, default BLAS threads)
        sub = np.ascontiguousarray(S[:, :cols])
        t0 = time.perf_counter()
        orc.dense_joint(y, src, v_s, sub, workers=1, K=K, W=W)
        t1 = time.perf_counter() - t0
        out["default_setting"] = dict(value=cols / t1, unit=UNIT, workers=1, blas_threads="library default",
                                      sample=f"first {cols} cases, one run")
    return out


def cpu_model() -> str:
    """The host CPU model string (lscpu), stated beside the core count."""
    try:
        out = subprocess.check_output(["lscpu"], text=True, stderr=subprocess.DEVNULL)
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.CalledProcessError):
        pass
    return "unknown"


def run_reference():
    world, rank, _ = dist_env()
    if rank != 0:
        return
    model, loads, method, desc, _, _ = workload(ARGS.config, 0, host_tau=1 << 16)
    cores = os.cpu_count() or 1
    from threadpoolctl import threadpool_limits
    from oracle import tpf_oracle as orc
    y, src, v_s = model.admittance.y_dd, model.source_injection(), model.slack.v_s
    S = loads.values
    # bounded sample sized so the whole run stays within a few minutes
    probe = cpu_sample(model, loads, 3.0, cores)
    per_step = max(2.0, min(20.0, 150.0 / max(1, ARGS.steps + ARGS.warmup)))
    cols = int(min(S.shape[1], max(64, probe["value"] * per_step)))
    if method == "sparse":
        cols = min(cols, 1200)
    sub = np.ascontiguousarray(S[:, :cols])
    times = []
    for i in range(ARGS.warmup + ARGS.steps):
        t0 = time.perf_counter()
        if method == "dense":
            with threadpool_limits(limits=1, user_api="blas"):
                orc.dense_joint(y, src, v_s, sub, workers=cores)  # setup included, like bench.py:139-165
        else:
            orc.sparse_block(y, src, v_s, sub)
        if i >= ARGS.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = cols / t
    line = dict(impl="reference", metric=METRIC, value=value, unit=UNIT, n_gpus=world,
                steps=ARGS.steps, warmup=ARGS.warmup, ms_per_step=t * 1e3, higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype="c128", data="synthetic",
                config=dict(workload=desc, tau_sample=cols, method=method),
                cpu_baseline=dict(value=value, unit=UNIT, cores=cores, kind="port", cpu=cpu_model(),
                                  sample=f"first {cols} of {S.shape[1]} cases per step, oracle port of "
                                         f"tpflow.batch_solve_{method} incl. setup"),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.out, _ = self.proc.communicate()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        sm = [float(r[1]) for r in rows]
        load = [float(r[1]) for r in rows if float(r[3]) > 150.0] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return dict(sm_mhz=float(np.median(load)), sm_max_mhz=float(rows[0][2]), samples=len(rows),
                    reasons=sorted(reasons))


def traffic_from_profiles(kernel, tau):
    """DRAM bytes per launch from the committed ncu capture, scaled to this tau."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh).get(kernel, {})
    except (OSError, ValueError):
        return None
    if "dram_bytes_per_launch" not in d:
        return None
    return d["dram_bytes_per_launch"] * (tau / d["tau"]) if d.get("tau") else d["dram_bytes_per_launch"]


def run_ours():
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # TPF_BENCH_ONE_GPU=1 (plumbing check only): every rank on cuda:0 over gloo.
    # The ranks never wait on each other inside a kernel, only at the barriers.
    if os.environ.get("TPF_BENCH_ONE_GPU") == "1":
        local = 0
    if world > 1:
        if os.environ.get("TPF_BENCH_ONE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            # NCCL's init log on stderr (communicator size per rank: the driver's nranks check)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2403_04578_b200 import DenseOperator, SparseOperator, LoadMatrix, _capi
    from paper_2403_04578_b200 import batch_solve_dense, batch_solve_sparse, SolveOptions
    from paper_2403_04578_b200._device import residual_and_summary

    if ARGS.config == "c4":
        return run_c4(dev, world, rank, local)
    n_buses = CONFIGS[ARGS.config][0]
    full_tau = ARGS.tau or CONFIGS[ARGS.config][2]
    scenarios = ARGS.config == "c4"
    device_gen = scenarios or (n_buses - 1) * full_tau * 16 > HOST_GEN_LIMIT
    model, loads, method, desc, tau, lspec = workload(ARGS.config, rank, host_tau=(1 << 16) if device_gen else None)
    b = model.n_demand
    lib = _capi.load()
    peak_tf = ctypes_probe(lib)
    c64 = ARGS.dtype == "c64"
    edt = np.complex64 if c64 else None
    tdt = torch.complex64 if c64 else torch.complex128
    if c64 and method == "dense" and b > 104:
        raise SystemExit("bench: the dense complex64 twin covers b <= 104")
    # c64: FP32 cannot resolve tol = 1e-10 (DESIGN 4.3b); the c64 bar is tol 1e-6, residual 1e-3
    opts = SolveOptions(tolerance=1e-6, residual_tolerance=1e-3) if c64 else SolveOptions()
    op = DenseOperator(model, dev, dtype=edt) if method == "dense" else SparseOperator(model, dev, dtype=edt)
    if scenarios:
        from paper_2403_04578_b200 import GenSpec
        from paper_2403_04578_b200.synth import gen_scenarios_device
        # scenario batches of this rank: s = rank, rank + world, ... (seed 1000 + s), generated on the
        # device before the timed region (the reference's harness also excludes generation, bench.py:4-7)
        S_list = [gen_scenarios_device(model, tau, GenSpec(n_buses=n_buses, seed=1000 + rank + world * i),
                                       device=dev) for i in range(max(1, min(ARGS.steps, 4)))]
    elif device_gen:
        from paper_2403_04578_b200.synth import gen_scenarios_device
        S_list = [gen_scenarios_device(model, tau, lspec, device=dev)]
    else:
        S_list = [torch.from_numpy(loads.values).to(dev)]
    S_list = [Sk.to(tdt) for Sk in S_list]
    S = S_list[0]
    V = torch.empty((b, tau), dtype=tdt, device=dev)
    iters_list = [torch.empty(tau, dtype=torch.int32, device=dev) for _ in S_list]  # one per scenario batch
    iters = iters_list[0]
    stream = torch.cuda.current_stream(dev)
    csr = op.contract.csr_on(dev)  # device buffers reused by every step: a step only enqueues kernels
    post = (torch.empty(tau, dtype=torch.float64, device=dev), torch.empty(tau, dtype=torch.uint8, device=dev),
            torch.empty(2, dtype=torch.int32, device=dev))

    fused = method == "sparse"

    def step(ev=None, k=0):
        Sk, itk = S_list[k % len(S_list)], iters_list[k % len(S_list)]
        if ev:
            ev[0].record(stream)
        if fused:  # sparse: residual post-check fused into the solve kernel
            op.solve(Sk, opts, V=V, iters=itk, resid=post[0])
        else:
            op.solve(Sk, opts, V=V, iters=itk)
        if ev:
            ev[1].record(stream)
        return residual_and_summary(op.contract, Sk, V, itk, opts.residual_tolerance, dev, csr=csr, out=post,
                                    have_resid=fused)

    if world > 1:
        # N > 1: every step goes through the product's tau-sharding (shard.solve_sharded,
        # local=True: each rank's resident slice; the batch iteration count and slice
        # sizes all-gathered over NCCL, no data-path collective)
        from paper_2403_04578_b200.shard import solve_sharded
        from paper_2403_04578_b200.dense import finish
        one_step = step

        def sharded_fn(_model, Sk, _opts):
            k = next(i for i, x in enumerate(S_list) if x is Sk)  # by identity (tensor == is elementwise)
            resid_k, mask_k, summ_k = one_step(None, k)
            return finish(V, iters_list[k], resid_k, mask_k, summ_k, True)

        def step(ev=None, k=0):  # noqa: F811 -- the sharded step
            Sk = S_list[k % len(S_list)]
            if ev:
                ev[0].record(stream)
            res = solve_sharded(model, Sk, opts, solve_fn=sharded_fn, local=True, gather=False,
                                return_on_device=True)
            if ev:
                ev[1].record(stream)
            return (res.residuals, res.converged_mask,
                    torch.stack([torch.tensor(res.iterations, device=dev), res.converged_mask.sum()]))

    for _ in range(ARGS.warmup):
        step()
    torch.cuda.synchronize(dev)
    # kernel-only timing (roofline): eager steps with events around the solve
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(ARGS.steps)]
    for k in range(ARGS.steps):
        out = step(kev[k], k)
    torch.cuda.synchronize(dev)
    # the timed steps replay one CUDA graph of the whole step (solve + residual +
    # summary: the same kernels on the same buffers, no per-launch host cost);
    # several scenario batches (C4) or --no-graph: eager launches
    graph = None
    if ARGS.graph and len(S_list) == 1 and world == 1:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                out = step()
            graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as exc:  # noqa: BLE001 -- report and fall back to eager
            print(f"bench: graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graph = None
            torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0.record(stream)
        for k in range(ARGS.steps):
            if graph is not None:
                graph.replay()
            else:
                out = step(None, k)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    ms = t0.elapsed_time(t1)
    kms = float(np.mean([a.elapsed_time(c) for a, c in kev]))
    # algorithmic work per launch: mean over the timed steps of sum_j n_j
    sum_n = int(round(sum(int(iters_list[k % len(S_list)].sum().item()) for k in range(ARGS.steps)) / ARGS.steps))
    launches = sum(launches_per_step(method, op, tau, iters_list[k % len(S_list)]) for k in range(ARGS.steps))
    summ = out[2].cpu().numpy()
    if world > 1:
        t = torch.tensor([ms, kms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
        agg = torch.tensor([tau, sum_n, int(summ[1])], dtype=torch.int64, device=dev)
        dist.all_reduce(agg)
        total_cases = int(agg[0])
        converged_all = int(agg[2])
    else:
        total_cases = tau
        converged_all = int(summ[1])
    value = total_cases * ARGS.steps / (ms * 1e-3)

    if c64 and method == "dense":
        alg = 8.0 * b * b * sum_n
        achieved = alg / (kms * 1e-3) / 1e12
        peak32 = fp32_peak(local)
        roofline = dict(bound="fp32", pipe="FP32 FFMA (SIMT; no FP32-exact tensor-core path on sm_100a)",
                        achieved=achieved, peak=peak32, unit="TFLOP/s", frac=achieved / peak32,
                        traffic=traffic_from_profiles("dense_c64_kernel", tau),
                        kernel="dense_c64_kernel", kernel_ms=kms,
                        peak_source="nominal: SMs x 128 FP32 lanes x 2 flop x max SM clock",
                        algorithmic=f"8*b^2*sum(n_j) = {alg:.4e} flop per launch")
    elif method == "dense":
        alg = 8.0 * b * b * sum_n  # FLOP_alg = 8 b^2 sum_j n_j
        achieved = alg / (kms * 1e-3) / 1e12
        roofline = dict(bound="tensor", pipe="FP64 DMMA (mma.sync m8n8k4)", achieved=achieved, peak=peak_tf, unit="TFLOP/s",
                        frac=achieved / peak_tf if peak_tf else None,
                        traffic=traffic_from_profiles(dense_kernel_name(b, tau), tau),
                        kernel=dense_kernel_name(b, tau), kernel_ms=kms,
                        peak_source="measured in-run: DMMA-only probe (tpf_probe_fp64_tflops); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                        algorithmic=f"8*b^2*sum(n_j) = {alg:.4e} flop per launch",
                        executed=executed_dense(b, sum_n, kms, peak_tf))
    else:
        alg = 48.0 * b * sum_n  # BYTES_alg = 48 b sum_j n_j
        achieved = alg / (kms * 1e-3) / 1e9
        peak = measured_hbm()
        if c64:
            alg /= 2.0  # 8-byte complex64 elements
        roofline = dict(bound="hbm", achieved=achieved * (0.5 if c64 else 1.0), peak=peak, unit="GB/s",
                        frac=achieved * (0.5 if c64 else 1.0) / peak,
                        traffic=None if c64 else traffic_from_profiles(op.kernel, tau), kernel=op.kernel,
                        kernel_ms=kms, peak_source="MEASURED_PEAKS.json hbm_gbs",
                        algorithmic=f"48*b*sum(n_j) = {alg:.4e} bytes per launch",
                        compulsory=dict(bytes=32.0 * b * tau, gbs=32.0 * b * tau / (kms * 1e-3) / 1e9,
                                        frac=32.0 * b * tau / (kms * 1e-3) / 1e9 / peak,
                                        what="S read once + V written once"))

    shard_gather = None
    if world > 1:
        # the optional final gather of the sharded path: all_gather of every
        # rank's device-resident V / counts / residuals / mask over NCCL, checked on this slice
        torch.cuda.synchronize(dev)
        dist.barrier()
        g0 = time.perf_counter()
        full = solve_sharded(model, S_list[0], opts, solve_fn=sharded_fn, local=True, gather=True,
                             return_on_device=True)
        torch.cuda.synchronize(dev)
        g_s = time.perf_counter() - g0
        mine_ok = bool(torch.equal(full.values[:, rank * tau:(rank + 1) * tau].to(dev), V))
        shard_gather = dict(api="paper_2403_04578_b200.shard.solve_sharded(..., local=True, gather=True, "
                                "return_on_device=True)", backend=dist.get_backend(), wall_ms=g_s * 1e3,
                            gathered_cases=int(full.values.shape[1]), own_slice_bitwise=mine_ok,
                            gathered_bytes=int(full.values.numel() * 16))
        del full
    e2e = None
    if not ARGS.no_e2e:
        e2e = run_e2e(model, loads, method, dev, batch_solve_dense, batch_solve_sparse, LoadMatrix, world,
                      dtype=edt, opts=opts)
    sparse = None
    if ARGS.config == "c2" and not c64 and ARGS.sparse_half and not ARGS.tau:
        graph = None
        del S_list, S, V, post
        torch.cuda.empty_cache()
        sparse = sparse_half(dev, world, rank)

    cpu = None
    if rank == 0 and world == 1 and not ARGS.no_cpu_baseline:
        cpu = cpu_sample(model, loads, ARGS.cpu_seconds, os.cpu_count() or 1)

    if rank == 0:
        line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=ARGS.steps,
                    warmup=ARGS.warmup, ms_per_step=ms / ARGS.steps, higher_is_better=True,
                    scaling="weak", vs_baseline=None, dtype=ARGS.dtype, data="synthetic",
                    config=dict(workload=desc + (" [complex64 twin, tol 1e-6]" if c64 else ""), b=b, tau_per_gpu=tau, method=method,
                                loads="device generator (synth.gen_scenarios_device)" if device_gen
                                else "host generator, bit-identical to tpflow.gen_scenarios",
                                sum_iterations=sum_n, batch_iterations=int(summ[0]),
                                converged=converged_all,
                                l2="inputs (S, V: %.0f MB each) larger than the 126 MB L2" % (b * tau * 16 / 1e6),
                                step_launch="cuda graph replay" if graph is not None else "eager",
                                parallelism=f"tau-sharded x{world} (independent scenario batches)",
                                **({"c4_full_1000_scenarios_s_extrapolated": 1000 * tau / value} if scenarios else {})),
                    roofline=roofline, cpu_baseline=cpu, e2e=e2e,
                    **({"sparse": sparse} if sparse is not None else {}),
                    **({"shard_gather": shard_gather} if shard_gather is not None else {}),
                    gpu_launches=launches,
                    clocks=clk.summary())
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_c4(dev, world, rank, local):
    """Config C4: the whole probabilistic-PF pass (probabilistic.probabilistic_pf) over
    --scenarios scenario batches of 525,600 cases (1,000 by default), scenarios
    dealt round-robin over ranks: per scenario the device generator, the dense
    solve with residual post-check and summary, and the per-node |V| statistics,
    all inside the timed region (CUDA events, max over ranks; strong scaling: the
    total work is fixed).  One untimed warm-up pass of min(--warmup, 3) scenarios."""
    import torch
    import torch.distributed as dist
    from paper_2403_04578_b200 import GenSpec, build_network
    from paper_2403_04578_b200.probabilistic import probabilistic_pf
    n_buses, _, tau, scale, _, desc = CONFIGS["c4"]
    if ARGS.tau:
        tau = ARGS.tau
    model = build_network(GenSpec(n_buses=n_buses, seed=0, load_scale=scale))
    n_scen = ARGS.scenarios
    probabilistic_pf(model, max(1, min(ARGS.warmup, 3)) * world, tau, device=dev)
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        w0 = time.perf_counter()
        t0.record(stream)
        st = probabilistic_pf(model, n_scen, tau, device=dev)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - w0
    ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    value = n_scen * tau / (ms * 1e-3)
    if rank == 0:
        line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=n_scen, warmup=max(1, min(ARGS.warmup, 3)),
                    ms_per_step=ms / n_scen, higher_is_better=True, scaling="strong", vs_baseline=None,
                    dtype="c128", data="synthetic",
                    config=dict(workload=desc, b=model.n_demand, tau_per_scenario=tau, scenarios=n_scen,
                                cases=n_scen * tau, method="dense",
                                step="one scenario batch: device generation + solve + residual/summary + "
                                     "per-node |V| statistics (nothing copied to the host)",
                                parallelism=f"scenarios round-robin over {world} rank(s), statistics all-reduced",
                                pass_s=ms * 1e-3, pass_wall_s=wall),
                    result=dict(vmin_min=float(st.vmin.min()), vmean_mean=float(st.vmean.mean()),
                                vmax_max=float(st.vmax.max()), nonconverged=st.nonconverged,
                                max_iterations=st.max_iterations, sum_iterations=st.sum_iterations),
                    gpu_launches=5 * n_scen, clocks=clk.summary())  # solve, residual, summary, 2 x stats
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sparse_half(dev, world, rank):
    """The sparse half of the metric (BASELINE metric "dense+sparse TPF"): config C3
    (b=5,000 radial feeder, tau=525,600 per rank, device-generated loads, rank r>0
    seed 1000+r) through SparseOperator.solve (warp-per-subtree kernel, fused
    residual, node-major input in case-major chunks), device-timed over the same
    --steps after --warmup steps, max over ranks; e2e through
    batch_solve_sparse(model, LoadMatrix) on a 65,536-case host sample; the CPU
    port of the reference's SuperLU block path on a bounded sample (rank 0, N=1)."""
    import torch
    import torch.distributed as dist
    from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, SolveOptions, LoadMatrix
    from paper_2403_04578_b200 import batch_solve_sparse, gen_scenarios
    from paper_2403_04578_b200.synth import gen_scenarios_device
    n_buses, _, tau, scale, _, desc = CONFIGS["c3"]
    model = build_network(GenSpec(n_buses=n_buses, seed=0, load_scale=scale))
    lspec = GenSpec(n_buses=n_buses, seed=0 if rank == 0 else 1000 + rank, load_scale=scale)
    b = model.n_demand
    S = gen_scenarios_device(model, tau, lspec, device=dev)
    V = torch.empty_like(S)
    iters = torch.empty(tau, dtype=torch.int32, device=dev)
    resid = torch.empty(tau, dtype=torch.float64, device=dev)
    op = SparseOperator(model, dev)
    opts = SolveOptions()
    stream = torch.cuda.current_stream(dev)
    for _ in range(ARGS.warmup):
        op.solve(S, opts, V=V, iters=iters, resid=resid)
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0.record(stream)
    for _ in range(ARGS.steps):
        op.solve(S, opts, V=V, iters=iters, resid=resid)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / ARGS.steps
    sum_n = int(iters.sum().item())
    conv = int((resid < opts.residual_tolerance).sum().item())
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    del S, V
    torch.cuda.empty_cache()
    peak = measured_hbm()
    alg = 48.0 * b * sum_n
    gbs = alg / (ms * 1e-3) / 1e9
    out = dict(workload=desc, b=b, tau_per_gpu=tau, value=world * tau / (ms * 1e-3), unit=UNIT,
               ms_per_step=ms, kernel=op.kernel, sum_iterations=sum_n, converged=conv,
               launches_per_step=3 * -(-tau // 65536),
               timing="device (CUDA events, eager launches; per step: per 65,536-case chunk a transpose in, "
                      "the subtree kernel with the fused residual, a transpose out), max over ranks",
               roofline=dict(bound="hbm", achieved=gbs, peak=peak, unit="GB/s", frac=gbs / peak,
                             kernel=op.kernel, peak_source="MEASURED_PEAKS.json hbm_gbs",
                             algorithmic=f"48*b*sum(n_j) = {alg:.4e} bytes per step (SURVEY 8(d))",
                             traffic=traffic_from_profiles("sparse_subtree_kernel", tau),
                             compulsory=dict(bytes=32.0 * b * tau, gbs=32.0 * b * tau / (ms * 1e-3) / 1e9,
                                             what="S read once + V written once")))
    if not ARGS.no_e2e:
        n = 1 << 16
        host = gen_scenarios(model, n, lspec)
        pinned = LoadMatrix(torch.from_numpy(host.values).pin_memory().numpy())
        for _ in range(2):
            r = batch_solve_sparse(model, pinned, device=dev)
        ts = []
        for _ in range(max(1, min(ARGS.steps, 3))):
            t_0 = time.perf_counter()
            r = batch_solve_sparse(model, pinned, device=dev)
            torch.cuda.synchronize(dev)
            ts.append(time.perf_counter() - t_0)
        te = float(np.mean(ts))
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        out["e2e"] = dict(value=world * n / te, unit=UNIT, ms_per_step=te * 1e3, cases_per_step=n,
                          h2d_bytes_per_step=b * n * 16, d2h_bytes_per_step=b * n * 16 + n * 13,
                          api="paper_2403_04578_b200.batch_solve_sparse(model, LoadMatrix) incl. the SuperLU "
                              "factorization of Y_dd (one per call, as the reference)",
                          iterations=int(r.iterations))
        if rank == 0 and world == 1 and not ARGS.no_cpu_baseline:
            out["cpu_baseline"] = sparse_cpu_sample(model, host, min(ARGS.cpu_seconds, 10.0))
    return out


def sparse_cpu_sample(model, loads, seconds):
    """The oracle port of tpflow.batch_solve_sparse (block system + one SuperLU per
    batch, sparse.py:167-207) on the first columns of the sample, single-threaded."""
    from oracle import tpf_oracle as orc
    y, src, v_s = model.admittance.y_dd, model.source_injection(), model.slack.v_s
    S = loads.values

    def run(cols):
        sub = np.ascontiguousarray(S[:, :cols])
        t_0 = time.perf_counter()
        orc.sparse_block(y, src, v_s, sub)
        return time.perf_counter() - t_0

    dt = run(16)
    cols = int(min(1200, max(16, 16 * seconds / max(dt, 1e-6) / 2)))
    t = float(np.median([run(cols) for _ in range(2)]))
    return dict(value=cols / t, unit=UNIT, cores=1, kind="port",
                sample=f"first {cols} of {S.shape[1]} cases, oracle port of tpflow.batch_solve_sparse "
                       "(block system + SuperLU, setup included), median of 2; the reference's SuperLU "
                       "fails from tau ~1,800 (SURVEY 8(d))")


def dense_kernel_name(b, tau):
    """The kernel tpf_dense_fpi_c128 / the large path runs for this shape (tpf_dense.cu dispatch)."""
    if b > 104:
        return "gemm_kernel (large-b active set)"
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return "dense_fpi_kernel" if tau <= 2 * sms * 64 else "dense_ws_kernel"


LARGE_HANDOFF = 256  # tpf_dense_large.cu kPtMax: active cases at the persistent hand-off


def launches_per_step(method, op, tau, iters=None):
    """Our kernels per timed step: dense = solve + residual + summary; sparse =
    one tree launch per compact chunk (SparseOperator) + summary, or the
    general kernel + residual + summary."""
    if method == "dense":
        if op.b <= 104:
            return 3
        # b > 104: init, then (prep, 64-case GEMM, 32-case GEMM, compact,
        # step) per iteration of the device-side WHILE loop (while more than
        # LARGE_HANDOFF cases are active), the persistent kernel once,
        # residual + summary
        it = iters.cpu().numpy() if hasattr(iters, "cpu") else np.asarray(iters)
        loop = 0
        while loop < int(it.max()) and int((it > loop).sum()) > LARGE_HANDOFF:
            loop += 1
        return 1 + 5 * loop + 1 + 2
    from paper_2403_04578_b200.sparse import TREE_CHUNK
    if op.sub is not None:  # per 65,536-case chunk: transpose in, subtree kernel, transpose out; + summary
        return 3 * -(-tau // 65536) + 1
    if op.tree is not None:
        return (-(-tau // TREE_CHUNK) if tau > TREE_CHUNK else 1) + 1
    return 3


def executed_dense(b, sum_n, kms, peak_tf):
    """FP64 tensor work the default kernel actually issues: 3M complex GEMM (3
    real DMMAs per complex 8x8x4 block-product) in both kernels; b <= 104 on
    the padded 8*ceil(b/8) x 4*ceil(b/4) operator, b > 104 (tiled active-set
    kernel) counted on the unpadded b x b operator."""
    if b <= 104:
        flop = 6.0 * (8 * -(-b // 8)) * (4 * -(-b // 4)) * sum_n
        how = "3M: 6 * 8ceil(b/8) * 4ceil(b/4) * sum(n_j)"
    else:
        flop = 6.0 * b * b * sum_n
        how = "3M: 6 b^2 sum(n_j) (tile padding not counted)"
    tf = flop / (kms * 1e-3) / 1e12
    return dict(flop=flop, tflops=tf, frac=tf / peak_tf if peak_tf else None, formula=how)


def ctypes_probe(lib):
    import ctypes
    tf, ms = ctypes.c_double(), ctypes.c_double()
    rc = lib.tpf_probe_fp64_tflops(ctypes.byref(tf), ctypes.byref(ms))
    return tf.value if rc == 0 else None


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0  # B200_PROFILING.md fallback


def fp32_peak(local):
    """Nominal FP32 FFMA peak (TFLOP/s) at the GPU's max SM clock."""
    import torch
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    try:
        mhz = float(subprocess.check_output(["nvidia-smi", "-i", str(local), "--query-gpu=clocks.max.sm",
                                             "--format=csv,noheader,nounits"], text=True).split()[0])
    except (OSError, subprocess.CalledProcessError, ValueError, IndexError):
        mhz = 1965.0
    return sms * 128 * 2 * mhz * 1e6 / 1e12


def run_e2e(model, loads, method, dev, bsd, bss, LoadMatrix, world, dtype=None, opts=None):
    """Public API from host memory; H2D/D2H inside the timed region, and the
    per-call setup too: the dense K = -inv(Y_dd), W memo is cleared before every
    timed call (the reference computes them per call, dense.py:151-152; the
    sparse path factorizes Y_dd per call anyway).  Headline: the caller's array
    already page-locked; ``pageable``: the same call on an ordinary numpy array
    (the library page-locks it for the call)."""
    import torch
    import torch.distributed as dist
    from paper_2403_04578_b200 import dense as dense_mod
    vals = loads.values if dtype is None else np.ascontiguousarray(loads.values, dtype=dtype)  # caller's c64 data
    pinned = torch.from_numpy(vals).pin_memory()
    # complex64: the caller's complex64 array goes in as is (batch_solve_*(..., dtype=complex64))
    host = LoadMatrix(pinned.numpy()) if dtype is None else pinned.numpy()
    solver = bsd if method == "dense" else bss
    out = None
    kw = {} if dtype is None else dict(dtype=dtype, opts=opts)
    if ARGS.chunk_cases:
        kw["chunk_cases"] = ARGS.chunk_cases
    for _ in range(3):  # populate torch's pinned-host cache exactly as the timed loop uses it
        out = None
        out = solver(model, host, device=dev, **kw)
    out = None
    torch.cuda.synchronize(dev)

    def timed(arr):
        if world > 1:
            dist.barrier()
        ts = []
        o = solver(model, arr, device=dev, **kw)  # untimed warm-up: one-time pinned staging allocation
        torch.cuda.synchronize(dev)
        o = None
        for _ in range(max(1, ARGS.steps)):
            with dense_mod._KW_LOCK:
                dense_mod._KW_CACHE.clear()  # setup inside the timed call, as the reference's
            o = None  # the caller has consumed the previous result (its pinned block is reused)
            t0 = time.perf_counter()
            o = solver(model, arr, device=dev, **kw)
            torch.cuda.synchronize(dev)
            ts.append(time.perf_counter() - t0)
        t = float(np.mean(ts))
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt[0])
        return t, o

    t, out = timed(host)
    # the pageable leg last: registering an ordinary array for the call disturbs later calls
    pageable = LoadMatrix(np.array(vals)) if dtype is None else np.array(vals)
    tp, _ = timed(pageable)
    del pageable
    b, tau = loads.values.shape
    esz = 8 if dtype is not None and np.dtype(dtype) == np.complex64 else 16
    h2d, d2h = int(b * tau * esz), int(b * tau * esz + tau * (4 + 8 + 1))
    floor_ms = pcie_floor_ms(h2d, d2h, dev)
    return dict(value=world * tau / t, unit=UNIT, h2d_bytes_per_step=h2d, cases_per_step=tau,
                d2h_bytes_per_step=d2h,
                ms_per_step=t * 1e3, api=f"paper_2403_04578_b200.batch_solve_{method}(model, LoadMatrix)",
                setup="included every call: K = -inv(Y_dd), W (dense; tree-LU solves on the device for radial feeders with b >= 64, "
                      "host LAPACK otherwise) / the factorization of Y_dd (sparse)",
                iterations=int(out.iterations),
                pageable=dict(value=world * tau / tp, ms_per_step=tp * 1e3,
                              how="the same call on an ordinary (pageable) numpy array"),
                pcie_floor=dict(ms=floor_ms, frac=floor_ms / (t * 1e3),
                                how="copy-only: same H2D and D2H bytes, pinned host, one copy stream per "
                                    "direction running concurrently, no compute; frac = floor / e2e"))


def pcie_floor_ms(h2d: int, d2h: int, dev) -> float:
    """The e2e roofline: the step's H2D and D2H bytes moved concurrently with nothing else."""
    import torch
    hi = torch.empty(h2d, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(d2h, dtype=torch.uint8, pin_memory=True)
    di = torch.empty(h2d, dtype=torch.uint8, device=dev)
    do = torch.empty(d2h, dtype=torch.uint8, device=dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ts = []
    for i in range(4):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        with torch.cuda.stream(s_in):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s_out):
            ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize(dev)
        if i:
            ts.append(time.perf_counter() - t0)
    del hi, ho, di, do
    return float(np.min(ts)) * 1e3


if __name__ == "__main__":
    if ARGS.impl == "reference":
        run_reference()
    else:
        run_ours()
