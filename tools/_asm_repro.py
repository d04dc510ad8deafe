import sys, math, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import fem3d as F
from paper_2112_00087_b200.ddm_fem import SubdomainSchwarz
from paper_2112_00087_b200.rowblock import rcb_partition
N=int(sys.argv[1]); parts=int(sys.argv[2])
cav=F.build_cavity(N); om=2*math.pi*100; A=cav.matrix(om)
S=SubdomainSchwarz(A, rcb_partition(cav.coords(), parts), complex(2, om/340), cav.lx/cav.nx, P.SolverOptions(tol=1e-10))
for m in (30,0):
    r=S.solve(cav.b, tol=1e-8, max_outer=40, m=m); print(m, r.report.outer_iterations, r.report.converged, flush=True)
