#!/bin/bash
# K1-NV12 3 x 40 KiB (default build) vs 2 x 60 KiB stages (tools/libclipdetect_nv2x60k.so), layout 6, interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CLIPDETECT_LIB=tools/libclipdetect_nv2x60k.so timeout 600 python -m pytest tests/test_gpu_nv12.py -x -q > gpurun_out/pytest_nv2x60k.log 2>&1
for r in 1 2 3; do
  timeout 300 python tools/nv12_micro.py 6000 > gpurun_out/nvstage_3x40k_r$r.log 2>&1
  CLIPDETECT_LIB=tools/libclipdetect_nv2x60k.so timeout 300 python tools/nv12_micro.py 6000 > gpurun_out/nvstage_2x60k_r$r.log 2>&1
done
