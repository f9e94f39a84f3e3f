#!/bin/bash
# usage: scripts/build_variant.sh <name> <extra nvcc flags...>  -> paper_2410_01359_b200/libflashmask_<name>.so
name=$1; shift
d=/tmp/fmv_$name; mkdir -p $d
cd "$(dirname "$0")/.."
for f in fm_api fm_prep fm_fwd fm_fwd2 fm_bwd fm_dq fm_f32; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c paper_2410_01359_b200/csrc/$f.cu -o $d/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2410_01359_b200/libflashmask_$name.so $d/*.o
