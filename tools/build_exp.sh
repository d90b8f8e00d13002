#!/bin/bash
# Experiment builds of libclipdetect (tools only, never the product path):
#   noatom: codes computed, histogram atomics removed;  notable: hue-table loads
#   replaced by a stand-in;  both.  Used with CLIPDETECT_LIB=tools/libclipdetect_<v>.so
set -e
cd "$(dirname "$0")/../paper_2503_12964_b200/csrc"
SRC="hist.cu hist_nv12.cu cuts.cu merge.cu sample.cu api.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared"
nvcc $F -DCLIPDETECT_EXP_NO_ATOMS -o ../../tools/libclipdetect_noatom.so $SRC &
nvcc $F -DCLIPDETECT_EXP_NO_TABLE -o ../../tools/libclipdetect_notable.so $SRC &
nvcc $F -DCLIPDETECT_EXP_NO_ATOMS -DCLIPDETECT_EXP_NO_TABLE -o ../../tools/libclipdetect_noboth.so $SRC &
wait
