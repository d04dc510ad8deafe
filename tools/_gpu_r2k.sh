set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2k_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2k_bench_ref.json 2> gpurun_out/r2k_bench_ref.err
TTS=c3,c5 timeout 2400 python tools/configs_tts.py > gpurun_out/r2k_tts.txt 2>&1
cp profiles/r02_time_to_solution.json gpurun_out/r02_time_to_solution_c35.json 2>/dev/null
tail -3 gpurun_out/r2k_gputests.txt
