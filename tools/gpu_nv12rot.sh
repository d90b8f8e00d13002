#!/bin/bash
# K1-NV12: layout 2 (default) vs layout 2 with the rotated lane -> unit map (dir 5), interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_nv12.py -x -q > gpurun_out/pytest_nv12rot.log 2>&1
for r in 1 2 3; do
  for d in ${NV_DIRS:-2 5}; do
    CLIPDETECT_NV12_DIR=$d timeout 300 python tools/nv12_micro.py 6000 > gpurun_out/nv12rot_d${d}_r$r.log 2>&1
  done
done
