#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_nv12.py -x -q -k "every_code_layout" > gpurun_out/pytest_nv12b.log 2>&1
for r in 1 2; do for d in 2 4; do
  CLIPDETECT_NV12_DIR=$d timeout 300 python tools/nv12_micro.py > gpurun_out/nv12b_d${d}_r$r.log 2>&1
done; done
echo done >> gpurun_out/pytest_nv12b.log
