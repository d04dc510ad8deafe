timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:"k_spmv" --csv python bench.py --steps 1 --warmup 0 --no-ilu > gpurun_out/r3b_ncu_spmv.csv 2> gpurun_out/r3b_ncu.err
PROBE_CASES=ref2d:0.0017,ref2d:0.00076 PROBE_SOLVERS=bicgstab_l PROBE_MAXIT=20 timeout 600 python tools/probe_configs.py > gpurun_out/r3b_probe.txt 2>&1
cat gpurun_out/r3b_probe.txt
