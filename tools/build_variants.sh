#!/bin/bash
# Build compile-time variants of libgiftb200.so into _variants/ for A/B runs
# (select one with GIFT_LIB=_variants/lib_<name>.so).  Every source except
# bmt.cu is compiled once; each variant recompiles bmt.cu with its -D flags.
# Variants are TUNING builds (-DGIFT_TUNING): they read the GIFT_* environment
# knobs the sweep scripts set and carry the extra kernel instances (512-thread
# and double-buffered tiled kernels, 2-chunk row kernel); the product build
# takes options only through gift_ctx_set_option.
#   tools/build_variants.sh "name1:-DX=1 -DY=2" "name2:-DX=3" ...
set -eu
cd "$(dirname "$0")/.."
mkdir -p _variants/obj
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wno-deprecated-declarations -DGIFT_TUNING"
S=paper_2502_17632_b200/csrc
for f in abi build filter metrics plio bookshelf shard hf peer; do
  [ _variants/obj/$f.o -nt $S/$f.cu ] && [ _variants/obj/$f.o -nt $S/common.cuh ] || nvcc $F -c $S/$f.cu -o _variants/obj/$f.o &
done
wait
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  ( nvcc $F $defs -c $S/bmt.cu -o _variants/obj/bmt_$name.o &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/lib_$name.so _variants/obj/{abi,build,filter,metrics,plio,bookshelf,shard,hf,peer}.o _variants/obj/bmt_$name.o &&
    echo "built _variants/lib_$name.so" ) &
done
wait
