#!/bin/bash
# One gpurun call (round 2): GPU tests, the bench line, and the DRAM traffic of
# the timed launch pattern (ncu --cache-control none: caches keep their natural
# state between the serialised launches, so L2 reuse across launches shows).
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
fi
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
fi
if [ "${TRAFFIC:-1}" = "1" ]; then
timeout 900 ncu --cache-control none --clock-control none -k regex:gemv7 -s 144 -c 96 --csv \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
  --log-file gpurun_out/traffic_$TAG.csv python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>> gpurun_out/bench_$TAG.err
echo "traffic rc=$?" >> gpurun_out/bench_$TAG.err
fi
tail -1 gpurun_out/pytest_$TAG.log 2>/dev/null; tail -2 gpurun_out/bench_$TAG.err
