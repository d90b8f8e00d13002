#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K1_CFGS=0,4 timeout 300 python tools/k1_micro.py 6000 > gpurun_out/exp_base.log 2>&1
CLIPDETECT_LIB=tools/libclipdetect_noatom.so K1_CFGS=0,4 timeout 300 python tools/k1_micro.py 6000 > gpurun_out/exp_noatom.log 2>&1
K1_CFGS=4 python tools/k1_micro.py 2000 > gpurun_out/exp_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_hist -s 2 -c 1 -o gpurun_out/k1_cfg4 python tools/k1_micro.py 2000 > gpurun_out/ncu_cfg4.log 2>&1
echo done >> gpurun_out/ncu_cfg4.log
