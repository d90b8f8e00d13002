#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K1_VIDEO=c3 K1_CFGS=49,14,26,51,55,53 timeout 900 python tools/k1_ab.py 1800 5 > gpurun_out/k1_ab_c3.log 2>&1
K1_CFGS=49,14 timeout 600 python tools/k1_ab.py 18000 3 > gpurun_out/k1_ab_c2_again.log 2>&1
echo done >> gpurun_out/k1_ab_c3.log
