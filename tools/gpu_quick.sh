#!/bin/bash
# quick gpurun: build, K1 config sweep, parity tests under the given K1 config(s)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
K1_CFGS=${K1_CFGS:-0,4} timeout 300 python tools/k1_micro.py 6000 > gpurun_out/k1_micro.log 2>&1
for c in ${TEST_CFGS:-4}; do
  CLIPDETECT_K1_CFG=$c timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu_cfg$c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_cfg$c.log
done
