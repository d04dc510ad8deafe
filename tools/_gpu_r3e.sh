set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > gpurun_out/r3e_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err
timeout 600 python bench.py --mode rowblock --no-ilu --steps 2 --warmup 1 > gpurun_out/r3e_rowblock.json 2> gpurun_out/r3e_rowblock.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r3e_bench_ref.json 2> gpurun_out/r3e_bench_ref.err
tail -3 gpurun_out/r3e_tests.txt
