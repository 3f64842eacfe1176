#!/bin/bash
# A/B build of libsssp_cuda.so with the rejected bucket paths compiled in
# (-DSSSP_BUCKET_AB=1: bulk-copy/TMA push, 16-deep register push) into
# build_ab/libsssp_cuda.so; select it with SSSP_LIB=build_ab/libsssp_cuda.so
# and SSSP_PUSH_BULK=1 / SSSP_PUSH_DEPTH16=1.
set -e
cd "$(dirname "$0")/.."
C=paper_2504_03667_b200/csrc
mkdir -p build_ab
make -s -j8 -C $C OUT=$(pwd)/build_ab/libsssp_cuda.so \
  NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3,-pthread --expt-relaxed-constexpr -DSSSP_BUCKET_AB=1" \
  BUILD_DIR=$(pwd)/build_ab/obj
