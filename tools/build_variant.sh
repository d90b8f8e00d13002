# Build libclipdetect from another copy of csrc/ into tools/ab/<tag>.so (A/B only; not the product).
# usage: bash tools/build_variant.sh <tag> <csrc dir>
TAG=$1; SRC=$2; OUT=tools/ab; mkdir -p $OUT/obj_$TAG
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
for f in hist hist_nv12 cuts merge sample api; do nvcc $F -c -o $OUT/obj_$TAG/$f.o $SRC/$f.cu & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $OUT/$TAG.so $OUT/obj_$TAG/*.o
