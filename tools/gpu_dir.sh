#!/bin/bash
# direct-offset K1 variants (cfg 22-27) vs cfg14/21: parity over every config, micro-benchmarks
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_k1_config or binmap" > gpurun_out/pytest_dir.log 2>&1
K1_CFGS=14,22,24,28,29,30,31,26 timeout 500 python tools/k1_micro.py 6000 > gpurun_out/k1_micro_dir.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nv12.py -x -q > gpurun_out/pytest_nv12_dir.log 2>&1
CLIPDETECT_NV12_DIR=0 timeout 300 python tools/nv12_micro.py > gpurun_out/nv12_micro_old.log 2>&1
CLIPDETECT_NV12_DIR=1 timeout 300 python tools/nv12_micro.py > gpurun_out/nv12_micro_dir.log 2>&1
echo done >> gpurun_out/k1_micro_dir.log
