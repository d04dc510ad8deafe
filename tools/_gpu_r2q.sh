set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fem3d.py tests/test_gpu_sweep.py tests/test_gpu_ilu0.py -m gpu -q -p no:cacheprovider -k "gmres or bicgstab_l or ref_mode or config1 or GMRES" 2>&1 | tail -25 > gpurun_out/r2q_tests.txt
PROBE_CASES=ref2d:0.0017,ref2d:0.00076 PROBE_SOLVERS=gmres PROBE_MAXIT=300 timeout 600 python tools/probe_configs.py > gpurun_out/r2q_probe.txt 2>&1
PROBE_CASES=ref2d:0.0017 PROBE_SOLVERS=gmres PROBE_MAXIT=60 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:"k_g_" --csv python tools/probe_configs.py > gpurun_out/r2q_ncu_gmres.csv 2> gpurun_out/r2q_ncu.err
tail -3 gpurun_out/r2q_tests.txt
cat gpurun_out/r2q_probe.txt
