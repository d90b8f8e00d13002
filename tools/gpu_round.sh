#!/bin/bash
# gpurun call: build, GPU tests, smoke, bench, K1 micro, ncu launch list + full capture of K1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
if [ -z "$SKIP_TESTS" ]; then
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
timeout 900 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/k1_micro.py 6000 > gpurun_out/k1_micro.log 2>&1; echo "micro rc=$?" >> gpurun_out/k1_micro.log
kill $CLK
if [ -n "$NCU" ]; then
  P="python bench.py --frames 2000 --steps 2 --warmup 1 --no-e2e --no-cpu"
  $P > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
  $P > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_hist -s 1 -c 1 -o gpurun_out/k1_full $P > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_sample -s 1 -c 1 -o gpurun_out/k4_full $P > gpurun_out/ncu_k4.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_k4.log
fi
