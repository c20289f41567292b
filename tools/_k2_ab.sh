#!/bin/bash
# K2 A/B: in-tree vs ablib/libcagra_k2old.so (optimize seconds from knn_time)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c1_parity.py -x -q -k "optimize or build_graph or c1" 2>&1 | tail -2
for r in 1 2; do
  timeout 300 python tools/knn_time.py 2>&1 | tail -1 | sed "s/^/new /"
  CAGRA_LIB=$PWD/ablib/libcagra_k2old.so timeout 300 python tools/knn_time.py 2>&1 | tail -1 | sed "s/^/old /"
done
