#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K1_CFGS=14,32,35,42,43,44,45,46 timeout 600 python tools/k1_micro.py 6000 > gpurun_out/k1_micro_dir4.log 2>&1
K1_CFGS=32,35,42,43,44,45,46 timeout 600 python tools/k1_micro.py 6000 > gpurun_out/k1_micro_dir4b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_k1_config" > gpurun_out/pytest_dir4.log 2>&1
echo done >> gpurun_out/k1_micro_dir4.log
