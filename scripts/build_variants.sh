#!/bin/bash
# Build tuning variants of libwavecast_b200.so into paper_2309_10212_b200/variants/
# usage: scripts/build_variants.sh name1 "FLAGS1" name2 "FLAGS2" ...
set -e
cd "$(dirname "$0")/../paper_2309_10212_b200/csrc"
mkdir -p ../variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  rm -rf build_var/$name; mkdir -p build_var/$name
  pids=()
  for f in wc_prims wc_volume wc_engine wc_stage wc_capi; do
    nvcc $ARCH -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags \
      -c $f.cu -o build_var/$name/$f.o &
    pids+=($!)
  done
  for p in "${pids[@]}"; do wait $p; done
  nvcc $ARCH -shared -o ../variants/lib_$name.so build_var/$name/*.o -lcudart
  echo built variants/lib_$name.so
done
