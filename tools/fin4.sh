timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fem3d.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "gmres or fem" 2>&1 | tail -3
PROBE_CASES=ref2d:0.0017,fem:79 PROBE_SOLVERS=gmres PROBE_MAXIT=300 timeout 300 python tools/probe_configs.py 2>&1 | tail -2
