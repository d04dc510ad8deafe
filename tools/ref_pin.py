"""Pin the BASELINE configs to the unmodified reference (TEST INFRASTRUCTURE).

Runs the reference itself (oracle/_ref/libcavac_ref.so, compiled from
/root/reference/proj/core/src by oracle/Makefile) on the systems the bench and
the config parity tests use, and records for each run the SolveReport plus a
SHA-256 of the solution bytes in tests/golden/configs_ref.json.  The full
solutions go to tests/_big/<case>.npy (git-ignored, travels to the GPU box).

The systems are built with the oracle's C restatement of build_grid/assemble
(bitwise the reference's, tests/test_oracle.py), never with the product.

    OMP_NUM_THREADS=8 python tools/ref_pin.py [case ...]

Cases (BASELINE.json configs; f = frequency, beta = wall admittance):
  c1_<solver>_<tol>   configs[0] size: h=0.0075 (50,721 DOF), 13 Hz, beta 0
  c2_bicgstab_<tol>   configs[1]: h=0.0017 (994,755 DOF), 100 Hz, beta 0.01
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "fixtures", "configs_ref.json")
BIG = os.path.join(ROOT, "tests", "_big")

SYSTEMS = {
    "c1": dict(h=0.0075, f=13.0, beta=0.0),
    "c2": dict(h=0.0017, f=100.0, beta=0.01),
}


def system(name):
    s = SYSTEMS[name]
    g = O.build_grid(2.4, 1.2, s["h"], 0.4, 0.65, s["beta"])
    rp, ci, v, b = O.assemble(g, 2 * math.pi * s["f"], 340.0, np.ones(g.roof_size, np.complex128))
    return rp, ci, v, b


def cases():
    out = {}
    for solver in ("bicgstab", "bicgstab_l", "tfqmr"):
        for tol in (1e-8, 1e-12):
            out[f"c1_{solver}_{tol:.0e}"] = ("c1", solver, tol, 40000)
    out["c2_bicgstab_1e-08"] = ("c2", "bicgstab", 1e-8, 20000)
    out["c2_bicgstab_1e-12"] = ("c2", "bicgstab", 1e-12, 40000)
    out["c2_tfqmr_1e-12"] = ("c2", "tfqmr", 1e-12, 40000)
    return out


def main(argv):
    allc = cases()
    todo = argv or list(allc)
    os.makedirs(BIG, exist_ok=True)
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    cache = {}
    for name in todo:
        sysname, solver, tol, max_iter = allc[name]
        if sysname not in cache:
            cache[sysname] = system(sysname)
        rp, ci, v, b = cache[sysname]
        t = time.time()
        x, rep = O.ref_solve(solver, rp, ci, v, b, tol=tol, max_iter=max_iter, l=8, parallel=True)
        wall = time.time() - t
        np.save(os.path.join(BIG, name + ".npy"), x)
        db[name] = {
            "system": sysname, **SYSTEMS[sysname], "n": int(len(rp) - 1), "nnz": int(len(v)),
            "solver": solver, "tol": tol, "max_iter": max_iter, "l": 8,
            "iterations": rep.iterations, "converged": rep.converged, "breakdown": rep.breakdown,
            "final_relres": rep.final_relres.hex(), "true_relres": rep.true_relres.hex(),
            "x_sha256": hashlib.sha256(np.ascontiguousarray(x).view(np.uint8)).hexdigest(),
            "x_norm": float(np.linalg.norm(x)),
            "wall_s": round(wall, 2), "threads": int(O.ref().ref_omp_threads()),
        }
        print(name, db[name], flush=True)
        with open(OUT, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
