#!/bin/bash
# One gpurun call: GPU tests, bench (both arms), ncu launch list + full capture.
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu --timeout 500 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>> gpurun_out/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 80 -c 4 \
   -o gpurun_out/full_$TAG python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>> gpurun_out/bench_$TAG.err
tail -1 gpurun_out/pytest_$TAG.log; tail -3 gpurun_out/bench_$TAG.err
