#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c1_parity.py -x -q -k "knn or ground_truth or c1 or build_graph" 2>&1 | tail -2
for r in 1 2; do
  CAGRA_KNN_TRACE=1 timeout 300 python tools/knn_time.py 2>&1 | tail -2 | sed "s/^/new /"
  CAGRA_KNN_TRACE=1 CAGRA_LIB=$PWD/ablib/libcagra_sortlist.so timeout 300 python tools/knn_time.py 2>&1 | tail -2 | sed "s/^/sorted /"
done
