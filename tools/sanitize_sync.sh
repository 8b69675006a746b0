#!/bin/bash
# compute-sanitizer synccheck + racecheck on small GEMV / decode cases (run via gpurun).
run() { echo "== $1 $2 :: $3"; timeout 900 compute-sanitizer --tool $1 --print-limit 3 python -m pytest "$2" -k "$3" -x -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|hazard|Barrier|Invalid|error|at .*\.cu:|in .*kernel" | head -14; }
run synccheck tests/test_gpu_parity.py "tma_kernel_paths_vs_oracle and shape1"
run synccheck tests/test_gpu_parity.py "glu_epilogue"
run synccheck tests/test_gpu_parity.py "norm_epilogue"
run synccheck tests/test_decode_gpu.py "attention_decode_vs_fp32 or rms_residual"
run racecheck tests/test_gpu_parity.py "tma_kernel_paths_vs_oracle and shape1"
run racecheck tests/test_decode_gpu.py "attention_decode_vs_fp32"
