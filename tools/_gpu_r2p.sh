set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2p_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2p_bench_ref.json 2> gpurun_out/r2p_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:"k_bf|k_bi|k_spmv_s" -c 80 --csv python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r2p_ncu_bench.csv 2> gpurun_out/r2p_ncu.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r2p_launches.csv 2> gpurun_out/r2p_launches.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bi_b_s|k_bf_b" -s 40 -c 1 -o gpurun_out/r2p_bicg_b python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r2p_ncu_full.log 2>&1
timeout 1200 python tools/ref_converge.py > gpurun_out/r2p_ref_full.txt 2>&1
cp profiles/r02_ref_full_solve.json gpurun_out/ 2>/dev/null
timeout 1200 python tools/parity_configs.py --c2-ref > gpurun_out/r2p_parity.txt 2>&1
cp profiles/r02_parity_configs.json gpurun_out/r02_parity_configs.json
tail -3 gpurun_out/r2p_tests.txt
