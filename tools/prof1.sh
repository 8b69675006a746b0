set -u
mkdir -p gpurun_out
export LD_LIBRARY_PATH=paper_2402_10517_b200
tools/micro/hmma_rate > gpurun_out/hmma_rate.txt 2>&1
tools/kbench/kbench all 0 20 > gpurun_out/kbench_base.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 2 -c 1 -o gpurun_out/steady_k3 tools/kbench/kbench 28672x8192 3 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 2 -c 1 -o gpurun_out/steady_k5 tools/kbench/kbench 28672x8192 5 2 > /dev/null 2>&1
ls gpurun_out
