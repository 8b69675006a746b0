#!/bin/bash
# one gpurun call: tests, a short bench, and an ncu capture of the GEMV kernels
set -u
mkdir -p gpurun_out
TAG=${1:-x}
timeout 600 python -m pytest tests -q -m gpu -x --timeout 500 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 400 python bench.py --steps ${STEPS:-300} --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -c 6 \
   -o gpurun_out/prof_$TAG python tools/prof_gemv.py --bits ${BITS:-3,4,8} > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
fi
tail -2 gpurun_out/pytest_$TAG.log; tail -1 gpurun_out/bench_$TAG.err
