timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fem3d.py tests/test_gpu_sweep.py -m gpu -q -p no:cacheprovider -k "gmres or ref_mode or config1 or uniform" 2>&1 | tail -3
for k in 1 2 3; do GMRES_IT=300 timeout 120 python tools/gmres_repro.py 2>&1 | tail -1 | cut -c1-100; done
PROBE_CASES=ref2d:0.0017,ref2d:0.00076,fem:79 PROBE_SOLVERS=gmres PROBE_MAXIT=300 timeout 300 python tools/probe_configs.py 2>&1 | tail -3
