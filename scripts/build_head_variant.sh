#!/bin/bash
# Build libwavecast_b200.so from a git revision (default HEAD) into
# paper_2309_10212_b200/variants/lib_<name>.so, for A/B runs against the
# working tree (scripts/gpu_variants_args.sh).  usage: build_head_variant.sh [rev] [name]
set -e
rev=${1:-HEAD}; name=${2:-head}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2309_10212_b200/csrc include | tar -x -C "$tmp"
cd "$tmp/paper_2309_10212_b200/csrc"; mkdir -p bv
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in wc_prims wc_volume wc_engine wc_stage wc_capi; do
  nvcc $ARCH -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -c $f.cu -o bv/$f.o 2>/dev/null &
done
wait
mkdir -p "$root/paper_2309_10212_b200/variants"
nvcc $ARCH -shared -o "$root/paper_2309_10212_b200/variants/lib_$name.so" bv/*.o -lcudart
rm -rf "$tmp"
echo "built variants/lib_$name.so from $rev"
