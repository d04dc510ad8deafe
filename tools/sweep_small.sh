for g in 200 148 96 64 32; do echo "== CVK_MAX_CTAS=$g"; CVK_MAX_CTAS=$g PROBE_CASES=ref2d:0.0075,fem:29 PROBE_SOLVERS=bicgstab,tfqmr,gmres timeout 300 python tools/probe_configs.py; done
