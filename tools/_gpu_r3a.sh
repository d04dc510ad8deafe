set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_breakdowns.py tests/test_gpu_sweep.py tests/test_gpu_cocg.py -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/r3a_tests.txt
timeout 900 python bench.py --no-ilu > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:"k_bf|k_uniform" -c 40 --csv python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r3a_ncu_bench.csv 2> gpurun_out/r3a_ncu.err
PROBE_CASES=ref2d:0.0017,fem:79,ref2d:0.00076 PROBE_SOLVERS=bicgstab,tfqmr,gmres,cocg PROBE_MAXIT=300 timeout 600 python tools/probe_configs.py > gpurun_out/r3a_probe.txt 2>&1
cat gpurun_out/r3a_tests.txt gpurun_out/r3a_probe.txt
