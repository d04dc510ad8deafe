for v in default w0 default w0; do
  if [ $v = default ]; then L=""; else L=_variants/$v/libcavac_b200.so; fi
  echo "== $v"; CVK_LIB_PATH=$L PROBE_CASES=ref2d:0.0017 PROBE_SOLVERS=gmres PROBE_MAXIT=300 timeout 300 python tools/probe_configs.py 2>&1 | tail -1
done
CVK_LIB_PATH=_variants/w0/libcavac_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "gmres" 2>&1 | tail -2
