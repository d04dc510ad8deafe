timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "gmres or ref_mode or config1" 2>&1 | tail -5 > gpurun_out/r2t_tests.txt
for v in default g2 g3 g4 g5 gmq2 default; do
  if [ $v = default ]; then L=""; else L=_variants/$v/libcavac_b200.so; fi
  echo "== $v" >> gpurun_out/r2t_probe.txt
  CVK_LIB_PATH=$L PROBE_CASES=ref2d:0.0017,ref2d:0.00076 PROBE_SOLVERS=gmres PROBE_MAXIT=300 timeout 600 python tools/probe_configs.py >> gpurun_out/r2t_probe.txt 2>&1
done
cat gpurun_out/r2t_tests.txt gpurun_out/r2t_probe.txt
