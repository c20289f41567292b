#!/bin/bash
# batch-1 A/B: atomic claim + id-indexed bitmap (in-tree) vs plain-load marks
# (ablib/libcagra_noclaim.so), each with and without the id-indexed bitmap
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_cta or b1_visited" 2>&1 | tail -2
G="10,96;16,64;12,64;10,64"
for r in 1 2; do
  timeout 400 python tools/b1_check.py 1000000 500 "$G" 2>&1 | grep "b1_kernel=1" | sed "s/^/claim+direct /"
  CAGRA_B1_DIRECT=0 timeout 400 python tools/b1_check.py 1000000 500 "$G" 2>&1 | grep "b1_kernel=1" | sed "s/^/claim+hash /"
  CAGRA_LIB=$PWD/ablib/libcagra_noclaim.so timeout 400 python tools/b1_check.py 1000000 500 "$G" 2>&1 | grep "b1_kernel=1" | sed "s/^/noclaim+direct /"
  CAGRA_B1_DIRECT=0 CAGRA_LIB=$PWD/ablib/libcagra_noclaim.so timeout 400 python tools/b1_check.py 1000000 500 "$G" 2>&1 | grep "b1_kernel=1" | sed "s/^/noclaim+hash /"
done
