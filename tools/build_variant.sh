#!/bin/bash
# Development aid: rebuild the library with extra nvcc flags into
# tools/_build/libendor_<name>.so (load it with ENDOR_LIB=...).
#   tools/build_variant.sh gv6 -DENDOR_GV_STAGES=6 -DENDOR_GV_WIN=9216
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/tools/_build/var_$name
mkdir -p "$out"
objs=()
for src in scan expand extract fixtures gemv gemv_fused gemm_fused capi pipeline storage vcode; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr -I"$root/include" -I"$root/paper_2406_11674_b200/csrc" "$@" \
    -c "$root/paper_2406_11674_b200/csrc/$src.cu" -o "$out/$src.o" &
  objs+=("$out/$src.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/tools/_build/libendor_$name.so" "${objs[@]}" -lcudart -ldl -lpthread
echo "$root/tools/_build/libendor_$name.so"
