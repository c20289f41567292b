#!/bin/bash
# K1 A/B: in-tree build vs ablib/libcagra_$1.so, interleaved, 3 builds each
for r in 1 2; do
  timeout 300 python tools/knn_time.py 2>&1 | tail -2 | sed "s/^/new /"
  CAGRA_LIB=$PWD/ablib/libcagra_$1.so timeout 300 python tools/knn_time.py 2>&1 | tail -2 | sed "s/^/$1 /"
done
