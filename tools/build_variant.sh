#!/bin/bash
# Build an A/B variant of libcagra_b200.so with extra -D flags on search.cu:
#   tools/build_variant.sh NAME "-DCAGRA_X=1 ..."  ->  ablib/libcagra_NAME.so
set -e
cd "$(dirname "$0")/.."
make -s build/capi.o build/graph_opt.o build/knn_exact.o build/knn_tc.o build/merge.o >/dev/null
mkdir -p ablib/obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2308_15136_b200/csrc"
$NV $2 -c paper_2308_15136_b200/csrc/search.cu -o ablib/obj/search_$1.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ablib/libcagra_$1.so \
  build/capi.o build/graph_opt.o build/knn_exact.o build/knn_tc.o build/merge.o ablib/obj/search_$1.o \
  -Xlinker -rpath -Xlinker /usr/local/cuda/lib64
