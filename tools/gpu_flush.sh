#!/bin/bash
# A/B of the K1 frame flush: default vs flush2 (two barriers, global RED per code)
# vs noflush (bound), alternating processes, C2 and C3 videos.
mkdir -p gpurun_out/flush
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/flush/build.log 2>&1
for r in 1 2; do
  for v in default flush2 noflush; do
    for vid in c2 c3; do
      if [ $v = default ]; then L=""; else L="CLIPDETECT_LIB=tools/libclipdetect_$v.so"; fi
      env $L K1_VIDEO=$vid K1_CFGS=55 timeout 300 python tools/k1_ab.py 18000 3 \
        > gpurun_out/flush/${v}_${vid}_r$r.log 2>&1
    done
  done
done
