#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K1_CFGS=14,32,35,42,45,26,37 timeout 900 python tools/k1_ab.py 18000 3 > gpurun_out/k1_ab1.log 2>&1
echo done >> gpurun_out/k1_ab1.log
