timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_breakdowns.py tests/test_gpu_cocg.py tests/test_gpu_sweep.py tests/test_gpu_fem3d.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
PROBE_CASES=ref2d:0.0017 PROBE_SOLVERS=bicgstab,cocg,tfqmr PROBE_MAXIT=2000 timeout 300 python tools/probe_configs.py 2>&1 | tail -3 | cut -c1-100
timeout 900 python bench.py > gpurun_out/fin6_bench.json 2> gpurun_out/fin6_bench.err
