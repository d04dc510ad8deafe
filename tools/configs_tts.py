"""Time to solution on every BASELINE.json config that fits one GPU.
Writes profiles/r02_time_to_solution.json (one section per config).

    TTS=c1,c2,c3,c5 python tools/configs_tts.py

c1  configs[0]: ~50k DOF, one frequency, GMRES(30) + Jacobi "as the reference
    runs it" -- the reference has no GMRES (krylov.cpp:377-384), so every
    solver runs: the reference's three, GMRES(30) and COCG; REF-2D cavity
    (h = 0.0075, 13 Hz) and the FEM-3D cavity (N = 29, 53,100 DOF).
c2  configs[1]: the 1M-DOF damped cavity (h = 0.0017, beta = 0.01) swept over
    50-500 Hz with the matrix resident (sweep.py), bench_solvers-style rows
    (pipeline.cpp:227-293): iterations / converged / device seconds per point
    for BiCGSTAB, BiCGSTAB(8), tfQMR, GMRES(30), COCG; fixed budget per point.
c3  configs[2]: ~5M DOF, 8 subdomains on one GPU: the reference's strip DDM
    (h = 0.00076, s = 2 + ik) with warm-started inner solves and the Krylov
    interface iteration, and the FEM-3D cavity (N = 135, 5M DOF) on 8 RCB
    subdomains (cvk_asm, FGMRES(30)); sweeps to converge and device time.
c5  configs[4]: ~50M DOF REF-2D (h = 0.00024) at a raised frequency: BiCGSTAB
    to 1e-8 and GMRES(30) for a fixed number of restarts (per-step cost).
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as H  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "r02_time_to_solution.json")
res = json.load(open(OUT)) if os.path.exists(OUT) else {}


def save():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    json.dump(res, open(OUT, "w"), indent=1)


def rep_row(r, extra=None):
    row = {"iterations": r.report.iterations, "converged": r.report.converged,
           "breakdown": r.report.breakdown, "final_relres": r.report.final_relres,
           "true_relres": r.report.true_relres, "device_s": r.report.device_time}
    row.update(extra or {})
    return row


SOLVERS = [("bicgstab", {}), ("bicgstab_l", {"l": 8}), ("tfqmr", {}), ("gmres", {"m": 30}), ("cocg", {})]
if os.environ.get("TTS_SOLVERS"):  # re-measure some solvers, keep the other rows
    SOLVERS = [sv for sv in SOLVERS if sv[0] in os.environ["TTS_SOLVERS"].split(",")]


def cavity(h, f, beta):
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, beta)
    return g, H.assemble(g, 2 * math.pi * f, 340.0, np.ones(g.roof_size(), np.complex128))


def c1():
    from paper_2112_00087_b200 import fem3d as F
    out = {}
    g, p = cavity(0.0075, 13.0, 0.0)
    cav = F.build_cavity(29)
    om = 2 * math.pi * 100.0
    for name, (A, b) in (("ref2d_h0.0075_13Hz", (p.A, p.b)), ("fem3d_N29_100Hz", (cav.matrix(om), cav.b))):
        M = P.jacobi(A)
        rows = {}
        for s, kw in SOLVERS:
            opts = P.SolverOptions(tol=1e-8, max_iter=200000, **kw)
            P.solve(P.solver_id(s), A, b, M, opts)  # warm-up
            r = P.solve(P.solver_id(s), A, b, M, opts)
            rows[s] = rep_row(r)
            print("c1", name, s, rows[s], flush=True)
        out[name] = {"n": A.nrows, "nnz": A.nnz(), "tol": 1e-8, "solvers": rows}
    res["c1"] = out
    save()


def c2():
    from paper_2112_00087_b200.sweep import frequency_sweep
    g = H.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
    freqs = [50.0 * k for k in range(1, 11)]
    out = {"n": g.size(), "tol": 1e-8, "budget": "max_iter 20000 (BiCGSTAB, tfQMR, COCG), 3000 cycles "
           "(BiCGSTAB(8)), 200000 Arnoldi steps (GMRES(30))", "rows": []}
    keep = {sv[0] for sv in SOLVERS}
    out["rows"] = [r for r in res.get("c2", {}).get("rows", []) if r["solver"] not in keep]
    budget = {"bicgstab": 20000, "bicgstab_l": 3000, "tfqmr": 20000, "gmres": 200000, "cocg": 40000}
    for s, kw in SOLVERS:
        t = frequency_sweep(g, 340.0, np.ones(g.roof_size(), np.complex128), freqs, solver=s,
                            opts=P.SolverOptions(tol=1e-8, max_iter=budget[s], **kw))
        for row in t.rows:
            d = {"solver": s, "frequency_hz": row.frequency_hz, "iterations": row.iterations,
                 "converged": row.converged, "breakdown": row.breakdown, "true_relres": row.true_relres,
                 "device_s": row.device_time_s, "point_s": row.point_time_s}
            out["rows"].append(d)
            print("c2", d, flush=True)
        res["c2"] = out
        save()


def c3():
    out = {}
    # the reference's strip DDM at 5M DOF, 8 strips
    from paper_2112_00087_b200 import schwarz as S
    from paper_2112_00087_b200.ddm_krylov import schwarz_solve_krylov
    g, p = cavity(0.00076, 13.0, 0.0)
    k = 2 * math.pi * 13.0 / 340.0
    part = S.partition(g, 8)
    tp = S.TransmissionParams(complex(2.0, k), complex(2.0, k))
    inner = P.SolverOptions(tol=1e-10)
    t = time.time()
    kr = schwarz_solve_krylov(p, part, tp, inner, tol=1e-8, max_sweeps=int(os.environ.get("TTS_C3_SWEEPS", "400")))
    import dataclasses
    d = {k: v for k, v in dataclasses.asdict(kr.report).items() if k != "residual_history"}
    d.update(n=g.size(), wall_s=time.time() - t, final_interface_residual=kr.report.residual_history[-1])
    out["ref2d_strips8_krylov"] = d
    print("c3", out, flush=True)
    res["c3"] = out
    save()
    # FEM-3D 5M DOF on 8 RCB subdomains (cvk_asm, FGMRES(30))
    from paper_2112_00087_b200 import fem3d as F
    from paper_2112_00087_b200.ddm_fem import SubdomainSchwarz
    from paper_2112_00087_b200.rowblock import rcb_partition
    cav = F.build_cavity(int(os.environ.get("TTS_C3_N", "135")))
    om = 2 * math.pi * 100.0
    A = cav.matrix(om)
    t = time.time()
    Sd = SubdomainSchwarz(A, rcb_partition(cav.coords(), 8), complex(2.0, om / 340.0), cav.lx / cav.nx,
                          P.SolverOptions(tol=1e-10))
    setup = time.time() - t
    r = Sd.solve(cav.b, tol=1e-8, max_outer=200, m=30)
    Sd.close()
    M = P.jacobi(A)
    mono = P.bicgstab(A, cav.b, M, P.SolverOptions(tol=1e-8, max_iter=100000))
    out["fem3d_rcb8_fgmres"] = {"n": A.nrows, "nnz": A.nnz(), "sweeps": r.report.outer_iterations,
                                "converged": r.report.converged, "device_s": r.report.device_time,
                                "setup_s": setup, "monodomain_bicgstab": rep_row(mono),
                                "rel_diff_vs_monodomain": float(np.linalg.norm(r.x - mono.x) / np.linalg.norm(mono.x))}
    print("c3", out["fem3d_rcb8_fgmres"], flush=True)
    res["c3"] = out
    save()


def c5():
    h = float(os.environ.get("TTS_C5_H", "0.00024"))
    f = float(os.environ.get("TTS_C5_F", "500"))
    g, p = cavity(h, f, 0.01)
    A = p.A
    M = P.jacobi(A)
    out = {"n": A.nrows, "nnz": A.nnz(), "frequency_hz": f, "beta": 0.01,
           "kh": 2 * math.pi * f / 340.0 * h}
    r = P.bicgstab(A, p.b, M, P.SolverOptions(tol=1e-8, max_iter=int(os.environ.get("TTS_C5_ITERS", "60000"))))
    out["bicgstab"] = rep_row(r, {"seconds_per_iteration": r.report.device_time / max(1, r.report.iterations)})
    print("c5", out, flush=True)
    res["c5"] = out
    save()
    steps = int(os.environ.get("TTS_C5_GMRES_STEPS", "300"))
    r = P.gmres(A, p.b, M, P.SolverOptions(tol=1e-8, m=30, max_iter=steps))
    out["gmres30"] = rep_row(r, {"seconds_per_step": r.report.device_time / max(1, r.report.iterations)})
    r = P.cocg(A, p.b, M, P.SolverOptions(tol=1e-8, max_iter=int(os.environ.get("TTS_C5_ITERS", "60000"))))
    out["cocg"] = rep_row(r, {"seconds_per_iteration": r.report.device_time / max(1, r.report.iterations)})
    print("c5", out, flush=True)
    res["c5"] = out
    save()


if __name__ == "__main__":
    for c in os.environ.get("TTS", "c1,c2").split(","):
        globals()[c]()
