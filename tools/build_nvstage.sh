#!/bin/bash
# Experiment build (tools only): K1-NV12 with 30 KiB stages (R = floor(10240 / W) chroma
# rows: 8 at 720p, i.e. 1280 tiles = exactly 2 per lane of 20 warps).  CLIPDETECT_LIB=tools/libclipdetect_nv30k.so
set -e
cd "$(dirname "$0")/../paper_2503_12964_b200/csrc"
SRC="hist.cu hist_nv12.cu cuts.cu merge.cu sample.cu api.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
nvcc $F -DCLIPDETECT_NV_STAGE_BYTES=30720 -o ../../tools/libclipdetect_nv30k.so $SRC
