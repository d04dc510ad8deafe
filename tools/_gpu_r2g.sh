set -x
PROBE_N=10,29,79 timeout 1200 python tools/asm_probe.py > gpurun_out/r2g_asm.txt 2>&1
cp profiles/r02_asm_probe.json gpurun_out/ 2>/dev/null
CVK_LIB_PATH=_variants/trace/libcavac_b200.so timeout 300 python tools/trace_phase.py > gpurun_out/r2g_trace.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bi|k_spmv_s" -c 40 --csv python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r2g_ncu_bicg.csv 2> gpurun_out/r2g_ncu.err
tail -2 gpurun_out/r2g_asm.txt
