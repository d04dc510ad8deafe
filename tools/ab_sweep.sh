#!/bin/bash
# A/B the measurement variants in _variants/ against the in-tree library on one box.
cd "$(dirname "$0")/.."
export PROBE_SOLVERS=${PROBE_SOLVERS:-bicgstab,tfqmr}
echo "== in-tree"; timeout 300 python tools/sweep_phase.py
for v in _variants/*/; do
  echo "== $v"; CVK_LIB_PATH=$v/libcavac_b200.so timeout 300 python tools/sweep_phase.py
done
