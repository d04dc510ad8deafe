set -x
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_breakdowns.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider 2>&1 | tail -6; done > gpurun_out/r2o_tests.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_asm.py tests/test_gpu_cocg.py -m gpu -q -p no:cacheprovider 2>&1 | tail -6 >> gpurun_out/r2o_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-ilu > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
CVK_LIB_PATH=_variants/trace/libcavac_b200.so timeout 300 python tools/trace_phase.py > gpurun_out/r2o_trace.txt 2>&1
cat gpurun_out/r2o_tests.txt | grep -E "passed|failed"
