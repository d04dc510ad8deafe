"""Timing and pinning probe of the reference-order device modes.

REF (ExecMode::Sequential) and REF_PAR (ExecMode::Parallel) must both give
the reference's iterates bit for bit; this prints their solve times on the
config-1 and config-2 systems and checks the SHA-256 of the solution against
tests/golden/configs_ref.json (the reference itself, tools/ref_pin.py).

    python tools/probe_refpar.py [c1|c2 ...]
"""
import hashlib
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

PIN = json.load(open(os.path.join(ROOT, "tests", "fixtures", "configs_ref.json")))


def system(name):
    s = PIN[[k for k in PIN if PIN[k]["system"] == name][0]]
    g = H.build_grid(2.4, 1.2, s["h"], 0.4, 0.65, s["beta"])
    p = H.assemble(g, 2 * math.pi * s["f"], 340.0, np.ones(g.roof_size(), np.complex128))
    return p.A, p.b


def main(which):
    for sysname in which:
        A, b = system(sysname)
        M = P.jacobi(A)
        for key, pin in sorted(PIN.items()):
            if pin["system"] != sysname:
                continue
            sid = P.solver_id(pin["solver"])
            opts = P.SolverOptions(tol=pin["tol"], max_iter=pin["max_iter"], l=pin["l"])
            modes = ["Parallel"] + (["Sequential"] if sysname == "c1" and pin["solver"] == "bicgstab" else [])
            for mode in modes:
                t = time.time()
                r = P.solve(sid, A, b, M, opts, mode=P.ExecMode[mode])
                wall = time.time() - t
                sha = hashlib.sha256(np.ascontiguousarray(r.x).view(np.uint8)).hexdigest()
                ok = (sha == pin["x_sha256"] and r.report.iterations == pin["iterations"]
                      and r.report.final_relres.hex() == pin["final_relres"])
                print(json.dumps({"case": key, "mode": mode, "bitwise_reference": ok,
                                  "iterations": r.report.iterations, "ref_iterations": pin["iterations"],
                                  "breakdown": r.report.breakdown, "device_s": round(r.report.device_time, 3),
                                  "wall_s": round(wall, 3), "ref_cpu_s": pin["wall_s"]}), flush=True)
            t = time.time()
            f = P.solve(sid, A, b, M, opts, mode=P.ExecMode.Fast)
            print(json.dumps({"case": key, "mode": "Fast", "iterations": f.report.iterations,
                              "breakdown": f.report.breakdown, "converged": f.report.converged,
                              "device_s": round(f.report.device_time, 4)}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1"])
