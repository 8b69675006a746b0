mkdir -p gpurun_out
for k in 3 8; do
ncu --set full --clock-control none --import-source on -k regex:gemv7 -s 2 -c 1 -o gpurun_out/v7a_k$k tools/kbench/kbench 28672x8192 $k 2 > gpurun_out/ncu_v7a_k$k.log 2>&1
done
timeout 300 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_v7a.log 2>&1; tail -3 gpurun_out/pytest_v7a.log
