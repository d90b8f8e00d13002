#!/bin/bash
# round-end evidence: GPU tests, smoke, RGB bench + ncu (launch list, K1 full), NV12 bench + ncu
mkdir -p gpurun_out
NCU=1 bash tools/gpu_round.sh
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_nv12.csv &
CLK=$!
timeout 900 python bench.py --format nv12 --steps 10 --warmup 3 > gpurun_out/bench_nv12.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_nv12.log
kill $CLK
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_nv12_kernel -s 2 -c 1 \
  -o gpurun_out/k1_nv12 python tools/nv12_micro.py 1000 > gpurun_out/ncu_nv12.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_nv12.log
