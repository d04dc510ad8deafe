set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/r2z_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
TTS=c1,c2 timeout 2400 python tools/configs_tts.py > gpurun_out/r2z_tts.txt 2>&1
cp profiles/r02_time_to_solution.json gpurun_out/r02_time_to_solution_final.json
tail -3 gpurun_out/r2z_tests.txt
