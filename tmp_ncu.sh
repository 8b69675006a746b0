mkdir -p gpurun_out
for k in 3 5; do
ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 2 -c 1 -o gpurun_out/v7i_k$k tools/kbench/kbench 28672x8192 $k 2 > gpurun_out/ncu_v7i_k$k.log 2>&1
done
