set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_asm.py tests/test_gpu_breakdowns.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2l_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-ilu > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
CVK_LIB_PATH=_variants/trace/libcavac_b200.so timeout 300 python tools/trace_phase.py > gpurun_out/r2l_trace.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:"k_bf|k_bi|k_spmv_s" -c 80 --csv python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r2l_ncu_bench.csv 2> gpurun_out/r2l_ncu.err
timeout 1200 python tools/ref_converge.py > gpurun_out/r2l_ref_full.txt 2>&1
cp profiles/r02_ref_full_solve.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/r2l_tests.txt
