#!/bin/bash
# A/B: product library (two-barrier flush) vs the previous three-barrier flush
# (tools/libclipdetect_oldflush.so, built from b1d4d18), alternating processes.
mkdir -p gpurun_out/flushab
for r in 1 2 3; do
  for v in default oldflush; do
    if [ $v = default ]; then L=""; else L="CLIPDETECT_LIB=tools/libclipdetect_$v.so"; fi
    env $L K1_VIDEO=c2 K1_CFGS=55 timeout 200 python tools/k1_ab.py 18000 3 > gpurun_out/flushab/${v}_c2_r$r.log 2>&1
  done
done
