#!/bin/bash
# Experiment builds of libclipdetect (tools only, never the product path):
#   noflush: frame flush only at the end of a CTA's range (wrong bins; bounds the flush cost)
#   flush2:  codes straight to the frame's global bins, two barriers per flush
# Used with CLIPDETECT_LIB=tools/libclipdetect_<v>.so
set -e
cd "$(dirname "$0")/../paper_2503_12964_b200/csrc"
SRC="hist.cu hist_nv12.cu cuts.cu merge.cu sample.cu api.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
nvcc $F -DCLIPDETECT_EXP_NO_FLUSH -o ../../tools/libclipdetect_noflush.so $SRC &
nvcc $F -DCLIPDETECT_EXP_FLUSH2 -o ../../tools/libclipdetect_flush2.so $SRC &
wait
