#!/bin/bash
# Round-2 evidence run (one gpurun call): GPU tests + smoke, bench (both arms),
# ncu launch list, ncu full captures (GEMV launches of the timed steps, one
# steady-state GEMV, one fused dense tcgen05 launch), DRAM traffic of the timed
# launch pattern (ncu --cache-control none).  Outputs under gpurun_out/ (TAG).
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
export LD_LIBRARY_PATH=paper_2402_10517_b200
timeout 1200 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>> gpurun_out/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 80 -c 4 \
   -o gpurun_out/full_$TAG python bench.py --profile --steps 2 --warmup 3 > /dev/null 2>> gpurun_out/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 2 -c 1 \
   -o gpurun_out/steady_k5_$TAG tools/kbench/kbench 28672x8192 5 2 > /dev/null 2>> gpurun_out/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_tc -s 2 -c 1 \
   -o gpurun_out/dense_$TAG python tools/dense_prof.py 512 > /dev/null 2>> gpurun_out/bench_$TAG.err
timeout 900 ncu --cache-control none --clock-control none -k regex:gemv7 -s 144 -c 96 --csv \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
  --log-file gpurun_out/traffic_$TAG.csv python bench.py --profile --steps 4 --warmup 3 > /dev/null 2>> gpurun_out/bench_$TAG.err
echo "all done" >> gpurun_out/bench_$TAG.err
tail -1 gpurun_out/pytest_$TAG.log; tail -3 gpurun_out/bench_$TAG.err
