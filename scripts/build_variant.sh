#!/bin/bash
# Build an A/B variant of libedbatch.so: scripts/build_variant.sh NAME -DFOO=1 ...  -> variants/libedbatch_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
SRC=${SRC:-paper_2302_03851_b200/csrc/ed_kernels.cu}
python -c "from paper_2302_03851_b200 import build as B; B.build()" > /dev/null
mkdir -p variants
B=paper_2302_03851_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2302_03851_b200/csrc "$@" \
  -c $SRC -o variants/k_$NAME.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libedbatch_$NAME.so variants/k_$NAME.o $B/ed_batch.cpp.o $B/ed_layout.cpp.o $B/ed_rl.cpp.o -lcudart_static -lrt -ldl -lpthread
rm -f variants/k_$NAME.o
echo variants/libedbatch_$NAME.so
