set -x
timeout 600 python -m pytest tests/test_gpu_asm.py tests/test_gpu_cocg.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/r2e_tests.txt
tail -3 gpurun_out/r2e_tests.txt
