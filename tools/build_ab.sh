#!/bin/bash
# Build search.cu A/B variants in parallel without make (the other objects
# must be current in build/):  tools/build_ab.sh NAME "FLAGS" [NAME "FLAGS" ...]
set -e
cd "$(dirname "$0")/.."
OBJS=$(for f in paper_2308_15136_b200/csrc/*.cu; do b=$(basename "$f" .cu); [ "$b" = search ] || echo "build/$b.o"; done)
mkdir -p ablib/obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2308_15136_b200/csrc"
while [ $# -ge 2 ]; do
  (
    $NV $2 -c paper_2308_15136_b200/csrc/search.cu -o ablib/obj/search_$1.o &&
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared \
      -o ablib/libcagra_$1.so $OBJS ablib/obj/search_$1.o -Xlinker -rpath -Xlinker /usr/local/cuda/lib64
  ) &
  shift 2
done
wait
