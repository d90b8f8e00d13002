#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K1_CFGS=55,49,59,60 timeout 900 python tools/k1_ab.py 18000 5 > gpurun_out/k1_ab7_c2.log 2>&1
K1_VIDEO=c3 K1_CFGS=55,49,59,60 timeout 900 python tools/k1_ab.py 1800 5 > gpurun_out/k1_ab7_c3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_k1_config" > gpurun_out/pytest_ab7.log 2>&1
echo done >> gpurun_out/k1_ab7_c2.log
