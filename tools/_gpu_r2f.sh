set -x
timeout 600 python -m pytest tests/test_gpu_asm.py tests/test_gpu_cocg.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2f_tests.txt
PROBE_N=10,29,79 timeout 900 python tools/asm_probe.py > gpurun_out/r2f_asm.txt 2>&1
cp profiles/r02_asm_probe.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/r2f_tests.txt
