set -x
timeout 600 python -m pytest tests/test_gpu_breakdowns.py tests/test_gpu_host_api.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2b_tests.txt
timeout 900 python tools/parity_configs.py --c2-ref > gpurun_out/r2b_parity.txt 2>&1
cp profiles/r02_parity_configs.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/r2b_tests.txt
