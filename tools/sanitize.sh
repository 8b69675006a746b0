#!/bin/bash
# compute-sanitizer memcheck over the kernel-level GPU tests (run via gpurun).
run() { echo "== $1 :: $2"; timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest "$1" -k "$2" -x -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds|Address|Program hit" | head -8; }
run tests/test_gpu_parity.py "tma_kernel_paths or glu_epilogue or norm_epilogue or dense_path or step_plan"
run tests/test_gpu_parity.py "small_batch or grouped_equals_single or pack_large"
run tests/test_decode_gpu.py "attention_decode_vs_fp32 or rms_residual or embed_rms or decode_step"
run tests/test_quant_gpu.py ""
run tests/test_fuzz_gpu.py ""
run tests/test_dist_fused_gpu.py "simulated"
run tests/test_apq_gpu.py ""
