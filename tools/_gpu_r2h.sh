set -x
PROBE_CYCLES=10 PROBE_REPS=2 timeout 300 python tools/bicgl_cycle.py > gpurun_out/r2h_bicgl_time.txt 2>&1
PROBE_CYCLES=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:k_bl -c 120 --csv python tools/bicgl_cycle.py > gpurun_out/r2h_ncu_bicgl.csv 2> gpurun_out/r2h_ncu_bicgl.err
PROBE_CYCLES=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bl_step --launch-skip 26 --launch-count 1 -o gpurun_out/r2h_bl_mgs -f python tools/bicgl_cycle.py > gpurun_out/r2h_ncu_full.txt 2>&1
PROBE_CYCLES=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bl_step --launch-skip 6 --launch-count 1 -o gpurun_out/r2h_bl_u3 -f python tools/bicgl_cycle.py >> gpurun_out/r2h_ncu_full.txt 2>&1
tail -3 gpurun_out/r2h_bicgl_time.txt
