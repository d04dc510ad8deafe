#!/bin/bash
# Drop-in check: the reference's own acceptance gate (proj/tests/acceptance.cpp)
# compiled with ITS non-solve modules (fvschemes, spectra, helmholtz, mmio,
# config, pipeline -- unmodified, straight from /root/reference) against this
# repo's cavac/{numkit,krylov,schwarz}.hpp and linked to the B200 library in
# place of the reference's numkit/krylov/schwarz.  Nothing is copied: the
# sources are compiled where they lie.  Output: dropin/_bin/acceptance_b200
# (git-ignored; it travels to the GPU box with the snapshot).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/dropin/_bin"
[ -d "$REF/core/src" ] || { echo "reference not present; skipping"; exit 0; }
mkdir -p "$OUT"
/usr/bin/g++ -std=c++20 -O2 -ffp-contract=off \
  -I"$ROOT/include" -I"$REF/core/include" \
  -DCAVAC_GOLDEN_DIR="\"tests/golden\"" \
  "$REF/tests/acceptance.cpp" \
  "$REF/core/src/fvschemes.cpp" "$REF/core/src/spectra.cpp" "$REF/core/src/helmholtz.cpp" \
  "$REF/core/src/mmio.cpp" "$REF/core/src/config.cpp" "$REF/core/src/pipeline.cpp" \
  "$ROOT/paper_2112_00087_b200/cpp/numkit_host.cpp" "$ROOT/paper_2112_00087_b200/cpp/krylov_host.cpp" \
  "$ROOT/paper_2112_00087_b200/cpp/schwarz_host.cpp" \
  -L"$ROOT/paper_2112_00087_b200" -lcavac_b200 -Wl,-rpath,'$ORIGIN/../../paper_2112_00087_b200' \
  -o "$OUT/acceptance_b200"
echo "$OUT/acceptance_b200"
