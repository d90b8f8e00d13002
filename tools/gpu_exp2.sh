#!/bin/bash
# what bounds the direct-offset K1: atomics / hue-table loads removed (experiment builds)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in default noatom notable noboth; do
  if [ $v = default ]; then
    K1_CFGS=14,32,35 timeout 300 python tools/k1_micro.py 4000 > gpurun_out/exp2_$v.log 2>&1
  else
    CLIPDETECT_LIB=tools/libclipdetect_$v.so K1_CFGS=14,32,35 timeout 300 python tools/k1_micro.py 4000 > gpurun_out/exp2_$v.log 2>&1
  fi
done
timeout 600 python -m pytest tests/test_gpu_nv12.py -x -q > gpurun_out/pytest_nv12_v.log 2>&1
for d in 0 1 2 3; do
  CLIPDETECT_NV12_DIR=$d timeout 300 python tools/nv12_micro.py > gpurun_out/nv12_micro_d$d.log 2>&1
done
echo done >> gpurun_out/exp2_default.log
