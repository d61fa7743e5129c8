#!/bin/bash
# Full A/B build (host planner + kernel with the same defines): scripts/build_full_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
D=/tmp/fv_$NAME; mkdir -p $D variants
C=paper_2302_03851_b200/csrc
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$C"
GX="g++ -O3 -std=c++17 -fPIC -ffp-contract=off -Iinclude -I$C -I/usr/local/cuda/include"
$NV "$@" -c $C/ed_kernels.cu -o $D/k.o &
$GX "$@" -c $C/ed_batch.cpp -o $D/b.o &
$GX "$@" -c $C/ed_layout.cpp -o $D/l.o &
$GX "$@" -c $C/ed_rl.cpp -o $D/r.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libedbatch_$NAME.so $D/k.o $D/b.o $D/l.o $D/r.o -lcudart_static -lrt -ldl -lpthread
echo variants/libedbatch_$NAME.so
