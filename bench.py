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
  e2e    the same solve the way a reference caller runs it (pipeline.cpp:196-202):
         cavac::jacobi + cavac::solve from a host CsrMatrix through the C++
         drop-in (libcavac_host.so), SolverOptions::fast_reductions -- per step
         the H2D of A (indices + values) and b and the D2H of x
  roofline  the solve's dominant kernels (the BiCGSTAB iteration) against
         the measured HBM copy peak: algorithmic bytes (40 nnz + 344 n per
         iteration) x iterations / device time
  cpu_baseline  the unmodified reference (oracle/_ref, ExecMode::Parallel,
         all host cores) timed on a bounded sample of the same solve

N > 1 (torchrun): one global BiCGSTAB over N row blocks, one per GPU
(rowblock.py / cvk_rowblock.cu; strong scaling).  Each rank assembles only its
own rows (helmholtz.assemble_rows), builds its plan from one all-gather of
halo lists (rowblock.plan_local_block) and its Jacobi from its own rows; the
reductions and halo values move in one NCCL all-gather per phase.  value is
the max over ranks.  --mode replicas keeps N independent copies.
--impl reference runs the reference CPU arm (oracle/_ref, never the product).
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
    """Identical in both arms (--impl b200 / reference)."""
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


def build_system_reference():
    """The same system from the oracle's restatement of build_grid/assemble
    (bitwise the reference's, tests/test_oracle.py): the reference arm never
    imports the product."""
    from oracle import oracle as O
    g = O.build_grid(2.4, 1.2, H, 0.4, 0.65, ADMITTANCE)
    return O.assemble(g, 2 * math.pi * FREQ_HZ, 340.0, np.ones(g.roof_size, np.complex128))


def uniform_offdiag(A):
    """True when every off-diagonal value of A is the same complex number bit
    for bit (the library then streams only the diagonal; cvk_blas.cu)."""
    rp = A.row_offsets.astype(np.int64)
    ci = A.col_indices.astype(np.int64)
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    off = A.values[ci != rows].view(np.uint64)
    return off.size > 0 and bool(np.all(off.reshape(-1, 2) == off.reshape(-1, 2)[0]))


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


def cpu_reference(system, steps, warmup, iters_full, sample_iters):
    """Time the unmodified reference (oracle/_ref) on a bounded sample;
    system = (rp, ci, v, b) as the reference assembles it."""
    from oracle import oracle as O
    rp, ci, v, b = system
    n = len(rp) - 1
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
        "sample": f"{sample_iters} BiCGSTAB iterations of the same {n}-DOF system "
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
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "replicas", "rowblock"],
                    help="auto: the single-device solve at N = 1, one global solve over N row blocks at "
                         "N > 1 (strong scaling); replicas: N independent copies of the solve")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="--mode rowblock: NCCL all-gathers, or the library's IPC mailbox exchange")
    ap.add_argument("--no-ilu", action="store_true", help="skip the ILU(0) side measurement")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.mode == "auto":
        args.mode = "single" if world == 1 else "rowblock"
    scaling = "weak" if args.mode == "replicas" else "strong"

    if args.impl == "reference":
        if rank != 0:
            return 0
        system = build_system_reference()
        iters_full = int(os.environ.get("CVK_REF_ITERS_FULL", str(REF_ITERS)))
        cb = cpu_reference(system, args.steps, args.warmup, iters_full, args.cpu_sample_iters)
        line = {
            "metric": METRIC, "value": cb["value"], "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["value"] * 1e3,
            "higher_is_better": False, "scaling": scaling, "vs_baseline": None, "dtype": "c128 (f64 complex)",
            "data": "synthetic (reference build_grid/assemble, roof Dirichlet 1+0i)", "impl": "reference",
            "config": workload_config(len(system[0]) - 1, len(system[2])),
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
    opts = _lib.CvkOpts(TOL, MAX_ITER, 8, 30, 0, _lib.MODE_FAST, 0, 0)
    torch.cuda.synchronize()

    def solve_device():
        rep = _lib.CvkReport()
        _lib.check(L.cvk_solve_device(dev.handle, 0, hA, hM, C.byref(opts), C.c_void_p(b_dev.data_ptr()),
                                      C.c_void_p(x_dev.data_ptr()), C.byref(rep)))
        return rep

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

    # end to end as a reference caller runs it: cavac::jacobi + cavac::solve
    # (pipeline.cpp:196-202) from a host CsrMatrix through the C++ drop-in
    e2e = e2e_dropin(A, prob.b, args.steps, barrier)
    t_e2e = e2e["seconds"]

    # SpMV GB/s (the metric's second number): the standalone streamed SpMV,
    # CUDA events on the library's stream, L2 flushed (256 MB write) before
    # every timed launch
    spmv_s = spmv_time(L, dev, hA, b_dev, reps=20)
    spmv_bytes = 20 * nnz + 4 * (n + 1) + 32 * n
    spmv_traffic = None  # ncu DRAM bytes of one k_spmv_s launch (profiles/r02_traffic.json)
    try:
        spmv_traffic = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json"))).get("spmv_dram_bytes")
    except Exception:
        pass

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
    # the streamed SpMV phases read 16 B of values per ROW when every
    # off-diagonal value is the same constant (CVK_OPT_UNIFORM_OFFDIAG, checked
    # on the device at each solve): the reference cavity's -c^2/h^2
    uniform = uniform_offdiag(A) and P.option("uniform_offdiag") != 0
    if uniform:
        iter_bytes = 8 * nnz + 376 * n  # 2 SpMVs of 4 nnz + 20 n instead of 20 nnz + 4 n
        setup_bytes = (16 * n * 4) + (20 * nnz + 4 * n + 48 * n) + (20 * nnz + 4 * n + 16 * n)  # + the check
        fmt = "CSR; off-diagonal values all equal (checked per solve): values streamed as the diagonal"
    else:
        iter_bytes = 40 * nnz + 344 * n
        setup_bytes = (16 * n * 4) + (20 * nnz + 4 * n + 48 * n)  # init pass + true residual
        fmt = "CSR"
    achieved = (iter_bytes * iters + setup_bytes) / t_solve / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bicgstab_iteration_dram_bytes")
        except Exception:
            traffic = None
    cb = cpu_reference((A.row_offsets.astype(np.int64), A.col_indices.astype(np.int64), A.values, prob.b),
                       1, 0, REF_ITERS, args.cpu_sample_iters)
    line = {
        "metric": METRIC,
        "value": t_solve, "unit": "s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_solve * 1e3, "higher_is_better": False, "scaling": scaling,
        "vs_baseline": None, "dtype": "c128 (f64 complex)",
        "data": "synthetic (reference build_grid/assemble, roof Dirichlet 1+0i)",
        "config": workload_config(n, nnz),
        "parallelism": "single GPU" if args.mode == "single" else f"replicas x{args.gpus}",
        "iterations": iters, "reference_iterations": REF_ITERS, "converged": bool(reps[-1].converged),
        "final_relres": reps[-1].final_relres, "true_relres": reps[-1].true_relres,
        "seconds_per_iteration": t_solve / max(iters, 1),
        "spmv": {"gbs": spmv_bytes / spmv_s / 1e9, "seconds": spmv_s,
                 "frac": spmv_bytes / spmv_s / 1e9 / peak, "bytes": spmv_bytes,
                 "timing": "CUDA events per launch on the library stream, L2 evicted by a 256 MB read before "
                           "each of 20 launches", "traffic": spmv_traffic},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "BiCGSTAB iteration: TMA-streamed SpMV phases k_bf_a_s + k_bf_b_s, "
                               "elementwise phase k_bf_c, reductions folded by the consumer "
                               "(3 launches per iteration, CUDA-graph replay)",
                     "matrix_format": fmt,
                     "traffic_unit": "DRAM bytes per iteration (ncu, sum of the 3 launches)",
                     "bytes_per_iteration": iter_bytes, "peak_kind": peak_kind},
        "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "path": "cavac::jacobi + cavac::solve (C++ drop-in, fast_reductions) from a host CsrMatrix",
                "iterations": e2e["iterations"], "device_s": e2e["device_s"]},
        "gpu_launches": launches,
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "clocks": clk.summary(),
        "x_finite": bool(np.isfinite(x_dev.cpu().numpy()).all()),
    }
    if ilu_side is not None:
        line["ilu0_side"] = ilu_side
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def e2e_dropin(A, b, steps, barrier):
    """cavac::jacobi + cavac::solve through dropin/_bin/libcavac_e2e.so
    (tools/dropin/e2e_shim.cpp over libcavac_host.so).  The host CsrMatrix is
    built once, as a reference caller already holds it; each timed call
    uploads A and b, solves, and downloads x."""
    lib = C.CDLL(os.path.join(ROOT, "dropin", "_bin", "libcavac_e2e.so"))
    lib.e2e_prepare.argtypes = [C.c_int64, C.c_int64] + [C.c_void_p] * 4
    lib.e2e_run.argtypes = [C.c_double, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
    n, nnz = A.nrows, A.nnz()
    rp = np.ascontiguousarray(A.row_offsets, np.uint64)
    ci = np.ascontiguousarray(A.col_indices, np.uint64)
    v = np.ascontiguousarray(A.values, np.complex128)
    bb = np.ascontiguousarray(b, np.complex128)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert lib.e2e_prepare(n, nnz, p(rp), p(ci), p(v), p(bb)) == 0
    x = np.zeros(n, np.complex128)
    out = np.zeros(5)
    assert lib.e2e_run(TOL, MAX_ITER, 1, p(x), p(out)) == 0  # warm-up (context, kernels)
    walls, devs = [], []
    for _ in range(max(1, steps)):
        barrier()
        assert lib.e2e_run(TOL, MAX_ITER, 1, p(x), p(out)) == 0
        walls.append(out[0])
        devs.append(out[1])
    return {"seconds": statistics.mean(walls), "device_s": statistics.mean(devs), "iterations": int(out[2]),
            "h2d": 8 * (n + 1) + 8 * nnz + 16 * nnz + 16 * n + 16 * n, "d2h": 16 * n}


def spmv_time(L, dev, hA, x_dev, reps=20):
    import torch
    st = torch.cuda.ExternalStream(L.cvk_ctx_stream(dev.handle))
    y = torch.empty_like(x_dev)
    # L2 (126 MB) evicted before every launch by READING a 256 MB buffer: a
    # write flush (round 2's first version) leaves L2 full of dirty lines whose
    # write-back then competes with the SpMV (34.8 vs 25.4 us in ncu)
    flush = torch.ones(32 << 20, dtype=torch.int64, device=x_dev.device)
    times = []
    with torch.cuda.stream(st):
        for k in range(reps + 2):
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            from paper_2112_00087_b200 import _lib
            _lib.check(L.cvk_spmv_device(hA, C.c_void_p(x_dev.data_ptr()), C.c_void_p(y.data_ptr()), 0))
            e1.record(st)
            e1.synchronize()
            if k >= 2:
                times.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.mean(times)


def run_rowblock(args, dist, world, rank, local):
    """One global BiCGSTAB over `world` row blocks, one per GPU (rowblock.py,
    csrc/cvk_rowblock.cu): strong scaling of the same system.  Setup is
    rank-local: each rank assembles its own rows (equal-row blocks of the
    cavity grid), derives its halo plan from one all-gather of halo lists and
    its Jacobi from its own diagonal.  value = device time of the solve (CUDA
    events on each rank's stream), max over ranks; e2e adds the per-step H2D
    of the rank's block and rhs (a fresh engine) and the D2H of its rows of x."""
    import torch
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import helmholtz as Hm
    from paper_2112_00087_b200.cavac import Device
    from paper_2112_00087_b200.rowblock import RowBlockEngine, local_jacobi, plan_local_block

    Device._default = Device(local)
    g = Hm.build_grid(2.4, 1.2, H, 0.4, 0.65, ADMITTANCE)
    n = g.size()
    bounds = np.array([(q * n) // world for q in range(world + 1)], np.int64)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    t_setup = time.perf_counter()
    rp, cols, vals, b_own = Hm.assemble_rows(g, 2 * math.pi * FREQ_HZ, 340.0, np.ones(g.roof_size(), np.complex128),
                                             r0, r1)

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    plan = plan_local_block(rank, bounds, rp, cols, vals, gather)
    d_own = local_jacobi(r0, rp, cols, vals)
    t_setup = time.perf_counter() - t_setup
    nnz_tot = int(sum(gather(len(vals))))
    opts = P.SolverOptions(tol=TOL, max_iter=MAX_ITER)
    eng = RowBlockEngine(plan, b_own, d_own, opts)

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
        e = RowBlockEngine(plan, b_own, d_own, opts)
        e.solve_p2p() if args.exchange == "p2p" else e.solve_nccl()
        x_own, rep = e.result()
        e.close()
        barrier()
        e2e.append(time.perf_counter() - t0)
    t = torch.tensor([t_solve, statistics.mean(e2e), t_setup], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_solve, t_e2e, t_setup = float(t[0]), float(t[1]), float(t[2])
    it = reps[-1].iterations
    if rank != 0:
        dist.destroy_process_group()
        return 0
    peak, peak_kind = peaks()
    iter_bytes = 40 * nnz_tot + 344 * n
    achieved = iter_bytes * it / t_solve / 1e9
    line = {
        "metric": METRIC, "value": t_solve, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_solve * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128 (f64 complex)",
        "data": "synthetic (reference build_grid/assemble, roof Dirichlet 1+0i)",
        "config": workload_config(n, nnz_tot),
        "parallelism": f"row blocks x{world} (one global BiCGSTAB, {args.exchange} exchange, rank-local setup)",
        "iterations": it, "reference_iterations": REF_ITERS, "converged": bool(reps[-1].converged),
        "final_relres": reps[-1].final_relres, "true_relres": reps[-1].true_relres,
        "seconds_per_iteration": t_solve / max(it, 1), "setup_s": t_setup,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                     "frac": achieved / (peak * world), "traffic": None,
                     "kernel": "row-block BiCGSTAB iteration (k_rb_a_s, k_rb_b_s, k_rb_c4, pack/post, "
                               "3 exchanges per iteration)", "bytes_per_iteration": iter_bytes,
                     "peak_kind": peak_kind + f" x {world} GPUs"},
        "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": 20 * nnz_tot + 48 * n,
                "d2h_bytes_per_step": 16 * n},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    print(json.dumps(line))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
