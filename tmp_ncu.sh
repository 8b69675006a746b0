mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 2 -c 1 -o gpurun_out/v7j_k3 tools/kbench/kbench 28672x8192 3 2 > /dev/null 2>&1
