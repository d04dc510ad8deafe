#!/bin/bash
# Build a measurement variant of libcavac_b200.so with extra nvcc defines:
#   tools/variant_build.sh <name> -DFOO ...   ->  _variants/<name>/libcavac_b200.so
# Select it at run time with CVK_LIB_PATH=_variants/<name>/libcavac_b200.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=_variants/$name
mkdir -p $out
objs=()
for src in paper_2112_00087_b200/csrc/*.cu; do
  f=$(basename $src .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude "$@" -c paper_2112_00087_b200/csrc/$f.cu -o $out/$f.o &
  objs+=($out/$f.o)
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libcavac_b200.so "${objs[@]}" -lcudart -ldl
rm -f "${objs[@]}"
echo $out/libcavac_b200.so
