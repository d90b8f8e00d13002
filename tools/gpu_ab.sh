#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_ab4.csv &
CLK=$!
K1_CFGS=14,49,51,53,54,55 timeout 900 python tools/k1_ab.py 18000 6 > gpurun_out/k1_ab4.log 2>&1
K1_CFGS=14,49,53 timeout 600 python tools/k1_ab.py 6000 4 > gpurun_out/k1_ab4_6000.log 2>&1
kill $CLK
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_k1_config" > gpurun_out/pytest_ab4.log 2>&1
echo done >> gpurun_out/k1_ab4.log
