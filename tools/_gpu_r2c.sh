set -x
timeout 300 python -m pytest tests/test_gpu_breakdowns.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2c_tests.txt
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2c_bench_ref.json 2> gpurun_out/r2c_bench_ref.err
timeout 600 python bench.py --mode rowblock --steps 2 --warmup 1 --no-ilu > gpurun_out/r2c_bench_rb.json 2> gpurun_out/r2c_bench_rb.err
timeout 600 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2c_bench_rb2.json 2> gpurun_out/r2c_bench_rb2.err
tail -2 gpurun_out/r2c_tests.txt
