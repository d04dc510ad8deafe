TTS=c2 TTS_SOLVERS=tfqmr timeout 900 python tools/configs_tts.py > gpurun_out/fin3_tts.txt 2>&1
cp profiles/r02_time_to_solution.json gpurun_out/r02_time_to_solution_tfqmr.json
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/fin3_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/fin3_bench.json 2> gpurun_out/fin3_bench.err
cat gpurun_out/fin3_tests.txt
