#!/usr/bin/env python3
"""Benchmark: complex-FP64 Helmholtz solve time to rel-res 1e-8 (+ SpMV GB/s).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
the reference's own 2-D cavity (build_grid(2.4, 1.2, h, 0.4, 0.65)) refined
to h = 0.0017 -> 1411 x 705 = 994,755 DOF, wall admittance beta = 0.01
(damping), one point of the 50-500 Hz sweep (f = 100 Hz), BiCGSTAB + Jacobi,
x0 = 0, tol = 1e-8 on the left-preconditioned relres (the reference's
criterion, krylov.hpp:46-49).  One step = one complete solve.

  value  device time of the solve with A, M, b resident in HBM (CUDA events
         on the solver's stream), max over ranks
  e2e    the same solve through the public C ABI from pinned host buffers:
         per step H2D of the frequency's matrix values + rhs, D2H of x
  roofline  the solve's dominant kernels (the BiCGSTAB iteration) against
         the measured HBM copy peak: algorithmic bytes (40 nnz + 344 n per
         iteration) x iterations / device time
  cpu_baseline  the unmodified reference (oracle/_ref, ExecMode::Parallel,
         all host cores) timed on a bounded sample of the same solve

N > 1 (torchrun): replicas -- every rank solves the same system on its own
GPU (the monodomain solve has no data-path exchange), value
is the max over ranks.  --impl reference runs the reference CPU arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "complex-FP64 solve time to rel-res 1e-8 and SpMV GB/s at 1/2/4/8 B200"
H = 0.0017
FREQ_HZ = 100.0
ADMITTANCE = 0.01
TOL = 1e-8
MAX_ITER = 20000
# the reference's own iteration count on this system (tools/ref_converge.py:
# oracle/_ref, ExecMode::Parallel, run to convergence: 6952 iterations, 688 s
# on 8 threads); the CPU baseline is its measured s/iteration x this count
REF_ITERS = 6952


def workload_config(n, nnz):
    return {
        "workload": "reference 2-D cavity (build_grid 2.4x1.2 m, roof 0.4-0.65) h=0.0017, "
                    "wall admittance 0.01, f=100 Hz of the 50-500 Hz sweep, BiCGSTAB + Jacobi, "
                    "tol 1e-8 (BASELINE.json configs[1])",
        "dof": n, "nnz": nnz, "solver": "bicgstab", "preconditioner": "jacobi",
        "tol": TOL, "frequency_hz": FREQ_HZ,
        "l2": "inputs larger than L2 (A 99 MB + 8 work vectors 127 MB > 126 MB L2)",
    }


def build_system():
    from paper_2112_00087_b200 import helmholtz as Hm
    g = Hm.build_grid(2.4, 1.2, H, 0.4, 0.65, ADMITTANCE)
    return Hm.assemble(g, 2 * math.pi * FREQ_HZ, 340.0, np.ones(g.roof_size(), np.complex128))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_reference(prob, steps, warmup, iters_full, sample_iters):
    """Time the unmodified reference (oracle/_ref) on a bounded sample."""
    from oracle import oracle as O
    A = prob.A
    rp, ci, v, b = (A.row_offsets.astype(np.int64), A.col_indices.astype(np.int64), A.values,
                    prob.b)
    if O.ref_available():
        kind = "reference"
        threads = O.ref().ref_omp_threads()

        def run():
            _, rep = O.ref_solve("bicgstab", rp, ci, v, b, tol=TOL, max_iter=sample_iters,
                                 parallel=True)
            return rep.wall_time
    else:
        kind = "port"
        threads = 1

        def run():
            _, rep = O.solve("bicgstab", rp, ci, v, b, tol=TOL, max_iter=sample_iters)
            return rep.wall_time
    for _ in range(max(0, warmup)):
        run()
    per_it = []
    for _ in range(max(1, steps)):
        per_it.append(run() / sample_iters)
    s_it = statistics.median(per_it)
    return {
        "value": s_it * iters_full, "unit": "s", "cores": threads, "kind": kind,
        "seconds_per_iteration": s_it,
        "sample": f"{sample_iters} BiCGSTAB iterations of the same {A.nrows}-DOF system "
                  f"(reference ExecMode::Parallel, OpenMP {threads} threads; dots single-threaded by "
                  f"the reference's design), median of {max(1, steps)}, extrapolated x {iters_full} "
                  f"iterations (the reference's own count on this system, tools/ref_converge.py)",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample-iters", type=int, default=40)
    ap.add_argument("--mode", default="replicas", choices=["replicas", "rowblock"],
                    help="N > 1: independent replicas (default), or one global solve over N row blocks "
                         "(rowblock.py, strong scaling)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="--mode rowblock: NCCL all-gathers, or the library's IPC mailbox exchange")
    ap.add_argument("--no-ilu", action="store_true", help="skip the ILU(0) side measurement")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        prob = build_system()
        iters_full = int(os.environ.get("CVK_REF_ITERS_FULL", str(REF_ITERS)))
        cb = cpu_reference(prob, args.steps, args.warmup, iters_full, args.cpu_sample_iters)
        line = {
            "metric": METRIC, "value": cb["value"], "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["value"] * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64 complex)",
            "data": "synthetic (reference build_grid/assemble)", "impl": "reference",
            "config": workload_config(prob.A.nrows, prob.A.nnz()),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return 0

    import torch
    dist = None
    if world > 1 or args.mode == "rowblock":
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    if args.mode == "rowblock":
        return run_rowblock(args, dist, world, rank, local)

    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import _lib
    from paper_2112_00087_b200.cavac import Device

    L = _lib.load()
    Device._default = Device(local)
    dev = Device._default
    prob = build_system()
    A = prob.A
    n, nnz = A.nrows, A.nnz()
    hA = A.device(dev)
    M = P.jacobi(A)
    hM = M.device(A, dev)

    b_dev = torch.from_numpy(prob.b.view(np.float64).copy()).to(f"cuda:{local}")
    x_dev = torch.zeros_like(b_dev)
    opts = _lib.CvkOpts(TOL, MAX_ITER, 8, 30, 0, _lib.MODE_FAST)
    torch.cuda.synchronize()

    def solve_device():
        rep = _lib.CvkReport()
        _lib.check(L.cvk_solve_device(dev.handle, 0, hA, hM, C.byref(opts), C.c_void_p(b_dev.data_ptr()),
                                      C.c_void_p(x_dev.data_ptr()), C.byref(rep)))
        return rep

    # pinned host buffers for the end-to-end leg
    vals_h = torch.from_numpy(A.values.view(np.float64).copy()).pin_memory()
    b_h = torch.from_numpy(prob.b.view(np.float64).copy()).pin_memory()
    x_h = torch.zeros_like(b_h).pin_memory()

    def solve_e2e():
        t0 = time.perf_counter()
        _lib.check(L.cvk_csr_set_values(hA, C.c_void_p(vals_h.data_ptr())))
        rep = _lib.CvkReport()
        _lib.check(L.cvk_solve(dev.handle, 0, hA, hM, C.byref(opts), C.c_void_p(b_h.data_ptr()),
                               C.c_void_p(x_h.data_ptr()), C.byref(rep)))
        return time.perf_counter() - t0, rep

    for _ in range(args.warmup):
        solve_device()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    launches = 0
    reps = []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            rep = solve_device()
            reps.append(rep)
            launches += int(rep.kernel_launches)
        barrier()
    dev_times = [r.device_time_s for r in reps]
    t_solve = statistics.mean(dev_times)
    iters = int(reps[-1].iterations)

    e2e_times = []
    barrier()
    for _ in range(args.steps):
        te, _r = solve_e2e()
        e2e_times.append(te)
    barrier()
    t_e2e = statistics.mean(e2e_times)
    x_check = x_h.numpy().view(np.complex128)

    # SpMV GB/s (standalone kernel, events, the metric's second number)
    ys = torch.empty_like(b_dev)
    spmv_s = C.c_double()
    _lib.check(L.cvk_spmv_bench(hA, C.c_void_p(b_dev.data_ptr()), C.c_void_p(ys.data_ptr()), 0, 50,
                                C.byref(spmv_s)))
    spmv_bytes = 20 * nnz + 4 * (n + 1) + 32 * n

    # beyond the reference: the same system with ILU(0) (3 sweeps per triangle)
    # instead of Jacobi -- a side number, not the headline (the reference has
    # no ILU(0); krylov.cpp:27-55)
    ilu_side = None
    if rank == 0 and not args.no_ilu:
        Mi = P.ilu0(A, 3)
        hMi = Mi.device(A, dev)
        ireps = []
        for k in range(2):
            rep = _lib.CvkReport()
            _lib.check(L.cvk_solve_device(dev.handle, 0, hA, hMi, C.byref(opts), C.c_void_p(b_dev.data_ptr()),
                                          C.c_void_p(x_dev.data_ptr()), C.byref(rep)))
            ireps.append(rep)
        r = ireps[-1]
        ilu_side = {"preconditioner": "ilu0 (exact factor, 3 Jacobi sweeps per triangle)",
                    "seconds": r.device_time_s, "iterations": int(r.iterations),
                    "converged": bool(r.converged), "true_relres": r.true_relres,
                    "seconds_per_iteration": r.device_time_s / max(1, r.iterations),
                    "speedup_vs_jacobi": t_solve / r.device_time_s if r.device_time_s > 0 else None,
                    "timing": "CUDA events around the solve (cvk_report.device_time_s), 1 warm-up"}
    if dist is not None:
        t = torch.tensor([t_solve, t_e2e], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_solve, t_e2e = float(t[0]), float(t[1])
    if rank != 0:
        dist.destroy_process_group()
        return 0

    peak, peak_kind = peaks()
    iter_bytes = 40 * nnz + 344 * n
    setup_bytes = (16 * n * 4) + (20 * nnz + 4 * n + 48 * n)  # init pass + true residual
    achieved = (iter_bytes * iters + setup_bytes) / t_solve / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bicgstab_iteration_dram_bytes")
        except Exception:
            traffic = None
    cb = cpu_reference(prob, 1, 0, REF_ITERS, args.cpu_sample_iters)
    line = {
        "metric": METRIC,
        "value": t_solve, "unit": "s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_solve * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (f64 complex)",
        "data": "synthetic (reference build_grid/assemble, roof Dirichlet 1+0i)",
        "config": dict(workload_config(n, nnz), parallelism=f"replicas x{args.gpus}"),
        "iterations": iters, "reference_iterations": REF_ITERS, "converged": bool(reps[-1].converged),
        "final_relres": reps[-1].final_relres, "true_relres": reps[-1].true_relres,
        "seconds_per_iteration": t_solve / max(iters, 1),
        "spmv": {"gbs": spmv_bytes / spmv_s.value / 1e9, "seconds": spmv_s.value,
                 "frac": spmv_bytes / spmv_s.value / 1e9 / peak, "bytes": spmv_bytes},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "BiCGSTAB iteration: TMA-streamed SpMV phases k_bi_a_s + k_bi_b_s, "
                               "elementwise phase k_bi_c (3 launches per iteration, CUDA-graph replay)",
                     "traffic_unit": "DRAM bytes per iteration (ncu, sum of the 3 launches)",
                     "bytes_per_iteration": iter_bytes, "peak_kind": peak_kind},
        "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": 16 * nnz + 16 * n,
                "d2h_bytes_per_step": 16 * n},
        "gpu_launches": launches,
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "clocks": clk.summary(),
        "x_finite": bool(np.isfinite(x_check).all()),
    }
    if ilu_side is not None:
        line["ilu0_side"] = ilu_side
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_rowblock(args, dist, world, rank, local):
    """One global BiCGSTAB over `world` row blocks, one per GPU (rowblock.py,
    csrc/cvk_rowblock.cu): strong scaling of the same system.  value = device
    time of the solve (CUDA events on each rank's stream), max over ranks;
    e2e adds the per-step H2D of the rank's matrix block and rhs (a fresh
    block) and the D2H of its rows of x."""
    import torch
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200.cavac import Device
    from paper_2112_00087_b200.rowblock import RowBlockEngine, plan_row_blocks

    Device._default = Device(local)
    prob = build_system()
    A = prob.A
    n, nnz = A.nrows, A.nnz()
    d = P.jacobi(A).inv_diag
    plan = plan_row_blocks(A, world)[rank]
    b = np.asarray(prob.b, np.complex128)
    opts = P.SolverOptions(tol=TOL, max_iter=MAX_ITER)
    eng = RowBlockEngine(plan, b[plan.r0:plan.r1], d[plan.r0:plan.r1], opts)

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    run = eng.solve_p2p if args.exchange == "p2p" else eng.solve_nccl
    for _ in range(args.warmup):
        run()
        eng.result()
    reps = []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            run()
            reps.append(eng.result()[1])
        barrier()
    t_solve = statistics.mean(r.device_time for r in reps)
    launches = sum(r.kernel_launches for r in reps)
    e2e = []
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        e = RowBlockEngine(plan, b[plan.r0:plan.r1], d[plan.r0:plan.r1], opts)
        e.solve_p2p() if args.exchange == "p2p" else e.solve_nccl()
        x_own, rep = e.result()
        e.close()
        barrier()
        e2e.append(time.perf_counter() - t0)
    t = torch.tensor([t_solve, statistics.mean(e2e)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_solve, t_e2e = float(t[0]), float(t[1])
    it = reps[-1].iterations
    if rank != 0:
        dist.destroy_process_group()
        return 0
    peak, peak_kind = peaks()
    iter_bytes = 40 * nnz + 344 * n
    achieved = iter_bytes * it / t_solve / 1e9
    line = {
        "metric": METRIC, "value": t_solve, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_solve * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128 (f64 complex)",
        "data": "synthetic (reference build_grid/assemble, roof Dirichlet 1+0i)",
        "config": dict(workload_config(n, nnz), parallelism=f"row blocks x{world} (one global BiCGSTAB)",
                       exchange=args.exchange),
        "iterations": it, "converged": bool(reps[-1].converged), "final_relres": reps[-1].final_relres,
        "true_relres": reps[-1].true_relres, "seconds_per_iteration": t_solve / max(it, 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                     "frac": achieved / (peak * world), "traffic": None,
                     "kernel": "row-block BiCGSTAB iteration (k_rb_a_s, k_rb_b_s, k_rb_c4, pack/post, "
                               "3 exchanges per iteration)", "bytes_per_iteration": iter_bytes,
                     "peak_kind": peak_kind + f" x {world} GPUs"},
        "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": 20 * nnz + 48 * n,
                "d2h_bytes_per_step": 16 * n},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    print(json.dumps(line))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
