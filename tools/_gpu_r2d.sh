set -x
timeout 600 python -m pytest tests/test_gpu_breakdowns.py tests/test_gpu_cocg.py tests/test_gpu_parity.py tests/test_gpu_host_api.py -m gpu -q -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/r2d_tests.txt
timeout 300 python tools/e2e_profile.py > gpurun_out/r2d_e2e_profile.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-ilu > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
tail -3 gpurun_out/r2d_tests.txt
