#!/bin/bash
# K1 A/B: cfg55 (default) vs cfg65 (4-deep ring of 640-group stages, 20 consumer warps)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_k1_config" > gpurun_out/pytest_ab${TAG:-9}.log 2>&1
K1_CFGS=${K1_CFGS:-55,65} timeout 900 python tools/k1_ab.py 18000 5 > gpurun_out/k1_ab${TAG:-9}_c2.log 2>&1
K1_VIDEO=c3 K1_CFGS=${K1_CFGS:-55,65} timeout 900 python tools/k1_ab.py 1800 5 > gpurun_out/k1_ab${TAG:-9}_c3.log 2>&1
