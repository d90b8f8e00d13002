#!/bin/bash
# NV12 check: build, NV12 parity tests, NV12 micro-benchmark (+ optional ncu capture)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_nv12.py -x -q ${PYTEST_ARGS} > gpurun_out/pytest_nv12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_nv12.log
timeout 300 python tools/nv12_micro.py ${NV12_FRAMES:-4000} > gpurun_out/nv12_micro.log 2>&1 || exit 0
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_nv12_kernel -s 2 -c 1 \
    -o gpurun_out/k1_nv12 python tools/nv12_micro.py 1000 > gpurun_out/ncu_nv12.log 2>&1
fi
