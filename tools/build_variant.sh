#!/bin/bash
# Build an A/B variant of libcagra_b200.so with extra -D flags on one source
# (default search.cu):
#   tools/build_variant.sh NAME "-DCAGRA_X=1 ..." [search_b1]  ->  ablib/libcagra_NAME.so
set -e
cd "$(dirname "$0")/.."
make -s paper_2308_15136_b200/lib/libcagra_b200.so >/dev/null
SRC=${3:-search}
# variants of search.cu: -DCAGRA_AB_HOT_ONLY keeps only the 96-d kernels (fast ptxas)
OBJS=$(for f in paper_2308_15136_b200/csrc/*.cu; do b=$(basename "$f" .cu); [ "$b" = "$SRC" ] || echo "build/$b.o"; done)
mkdir -p ablib/obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2308_15136_b200/csrc"
$NV $2 -c paper_2308_15136_b200/csrc/$SRC.cu -o ablib/obj/${SRC}_$1.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ablib/libcagra_$1.so \
  $OBJS ablib/obj/${SRC}_$1.o \
  -Xlinker -rpath -Xlinker /usr/local/cuda/lib64
