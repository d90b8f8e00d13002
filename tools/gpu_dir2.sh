#!/bin/bash
# hash variants of the direct-offset K1 + ncu of cfg14 vs cfg32 (shared-memory pipe metrics)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K1_CFGS=14,32,33,34,30,22 timeout 500 python tools/k1_micro.py 6000 > gpurun_out/k1_micro_dir2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_k1_config" > gpurun_out/pytest_dir2.log 2>&1
K1_CFGS=14,32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_hist -c 2 \
  -o gpurun_out/k1_dir2 python tools/k1_one.py 2000 > gpurun_out/ncu_dir2.log 2>&1
echo done >> gpurun_out/k1_micro_dir2.log
