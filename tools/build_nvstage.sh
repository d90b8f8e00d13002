#!/bin/bash
# Experiment builds (tools only) of K1-NV12 ring shapes; CLIPDETECT_LIB=tools/libclipdetect_<tag>.so
#   nv30k: 4 x 30 KiB (R = floor(10240 / W))   nv3x40k: 3 x 40 KiB (R = floor(13653 / W))
#   nv2x60k: 2 x 60 KiB (R = floor(20480 / W); now the default)
set -e
cd "$(dirname "$0")/../paper_2503_12964_b200/csrc"
SRC="hist.cu hist_nv12.cu cuts.cu merge.cu sample.cu api.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
case "${1:-nv3x40k}" in
  nv30k) nvcc $F -DCLIPDETECT_NV_STAGE_BYTES=30720 -o ../../tools/libclipdetect_nv30k.so $SRC ;;
  nv3x40k) nvcc $F -DCLIPDETECT_NV_STAGES=3 -DCLIPDETECT_NV_STAGE_BYTES=40960 -o ../../tools/libclipdetect_nv3x40k.so $SRC ;;
  nv2x60k) nvcc $F -DCLIPDETECT_NV_STAGES=2 -DCLIPDETECT_NV_STAGE_BYTES=61440 -o ../../tools/libclipdetect_nv2x60k.so $SRC ;;
esac
