#!/bin/bash
# Build an A/B variant of libcagra_b200.so with extra -D flags on search.cu:
#   tools/build_variant.sh NAME "-DCAGRA_X=1 ..."  ->  ablib/libcagra_NAME.so
set -e
cd "$(dirname "$0")/.."
make -s paper_2308_15136_b200/lib/libcagra_b200.so >/dev/null
OBJS=$(for f in paper_2308_15136_b200/csrc/*.cu; do b=$(basename "$f" .cu); [ "$b" = search ] || echo "build/$b.o"; done)
mkdir -p ablib/obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2308_15136_b200/csrc"
$NV $2 -c paper_2308_15136_b200/csrc/search.cu -o ablib/obj/search_$1.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ablib/libcagra_$1.so \
  $OBJS ablib/obj/search_$1.o \
  -Xlinker -rpath -Xlinker /usr/local/cuda/lib64
