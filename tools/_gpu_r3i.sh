timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cocg.py tests/test_gpu_breakdowns.py tests/test_gpu_configs.py tests/test_gpu_sweep.py tests/test_gpu_fem3d.py -m gpu -q -p no:cacheprovider 2>&1 | tail -6
PROBE_CASES=ref2d:0.0017,fem:79,ref2d:0.00076 PROBE_SOLVERS=cocg PROBE_MAXIT=2000 timeout 300 python tools/probe_configs.py 2>&1 | tail -3
