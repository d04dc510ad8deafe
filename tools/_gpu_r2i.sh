set -x
timeout 900 python -m pytest tests/test_gpu_ddm_dist.py tests/test_gpu_asm.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2i_tests.txt
bash tools/_gpu_r2h.sh
PROBE_N=10,29,79 timeout 1500 python tools/asm_probe.py > gpurun_out/r2i_asm.txt 2>&1
cp profiles/r02_asm_probe.json gpurun_out/ 2>/dev/null
TTS=c1,c2 timeout 2400 python tools/configs_tts.py > gpurun_out/r2i_tts.txt 2>&1
cp profiles/r02_time_to_solution.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/r2i_tests.txt
