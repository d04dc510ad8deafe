for v in default st5 st8 st3 default st5; do
  if [ $v = default ]; then L=""; else L=_variants/$v/libcavac_b200.so; fi
  echo "== $v"; CVK_LIB_PATH=$L PROBE_CASES=ref2d:0.0017,fem:79 PROBE_SOLVERS=bicgstab,cocg,tfqmr PROBE_MAXIT=2000 timeout 300 python tools/probe_configs.py 2>&1 | tail -6
done
