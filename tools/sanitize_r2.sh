#!/bin/bash
# compute-sanitizer over the round-2 kernels: the fused tcgen05 dense path
# (small / split-K / 256-wide tiles, k = 2..8) and the packer's code-range flag.
set -u
mkdir -p gpurun_out
export LD_LIBRARY_PATH=paper_2402_10517_b200
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 --error-exitcode 7 \
     python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider \
       -k "dense_tcgen05_vs_dense_oracle and 17 or split_k or pack_errors or cta_pair" > gpurun_out/san_r2_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_r2_$tool.log
  tail -3 gpurun_out/san_r2_$tool.log
done
