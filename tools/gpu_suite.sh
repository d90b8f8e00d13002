mkdir -p gpurun_out/r2
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke rc=$?
timeout 2700 python -m pytest tests -m gpu -q -rP -p no:cacheprovider --durations=15 > gpurun_out/r2/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2/pytest_gpu.log
timeout 600 python tools/k1_micro.py 6000 > gpurun_out/r2/k1_micro.log 2>&1; echo micro rc=$?
timeout 600 python tools/nv12_micro.py 6000 > gpurun_out/r2/nv12_micro.log 2>&1; echo nv12 rc=$?
cat gpurun_out/r2/k1_micro.log gpurun_out/r2/nv12_micro.log | tail -4
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench.log 2> gpurun_out/r2/bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/r2/bench.log
