#!/bin/bash
# build compile-time variants of the C-ABI library into tools/kbench/var_<name>/
# usage: variants.sh name "-DFOO=1 -DBAR=2" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/../.."
while [ $# -ge 2 ]; do
  d=tools/kbench/var_$1; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
     -o $d/libanyprec_b200.so paper_2402_10517_b200/csrc/*.cu &
  shift 2
done
wait
