set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_breakdowns.py -m gpu -q -p no:cacheprovider -k "bicgstab_l or breakdown or ref_mode or fast" 2>&1 | tail -5 > gpurun_out/r2j_tests.txt
PROBE_CYCLES=10 PROBE_REPS=2 timeout 300 python tools/bicgl_cycle.py > gpurun_out/r2j_bicgl_time.txt 2>&1
PROBE_CYCLES=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:k_bl -c 120 --csv python tools/bicgl_cycle.py > gpurun_out/r2j_ncu_bicgl.csv 2> gpurun_out/r2j_ncu_bicgl.err
tail -3 gpurun_out/r2j_tests.txt
cat gpurun_out/r2j_bicgl_time.txt
