#!/bin/bash
# phased-grid sweep: CTAs = multiple x occupancy x SMs (capped at #chunks)
for gm in 1 2 4 32; do
  echo "== CVK_PHASED_GRID=$gm"
  CVK_PHASED_GRID=$gm PROBE_SOLVE_S=1 PROBE_MAXIT=300 PROBE_SOLVERS=bicgstab,tfqmr python tools/probe.py 2>&1 | grep -E "bicgstab|tfqmr"
  CVK_PHASED_GRID=$gm PROBE_H=0.00054 PROBE_SOLVE_S=1 PROBE_MAXIT=60 PROBE_SOLVERS=bicgstab python tools/probe.py 2>&1 | grep -E "bicgstab"
done
