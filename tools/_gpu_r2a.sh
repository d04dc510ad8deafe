set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r2_gputests.txt
timeout 300 python tools/probe_refpar.py c1 > gpurun_out/r2_refpar_c1.txt 2>&1
timeout 300 python -c "
import sys,time,math; sys.path.insert(0,'.')
import numpy as np, paper_2112_00087_b200 as P
from paper_2112_00087_b200 import helmholtz as H
g=H.build_grid(2.4,1.2,0.0017,0.4,0.65,0.01); p=H.assemble(g,2*math.pi*100,340.0,np.ones(g.roof_size(),complex))
M=P.jacobi(p.A)
for mode in ('Parallel','Fast'):
  for it in (20,60):
    r=P.solve(0,p.A,p.b,M,P.SolverOptions(tol=1e-8,max_iter=it),mode=P.ExecMode[mode])
    print(mode,it,r.report.iterations,r.report.device_time, flush=True)
" > gpurun_out/r2_refpar_c2.txt 2>&1
tail -3 gpurun_out/r2_gputests.txt
