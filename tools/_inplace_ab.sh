#!/bin/bash
# in-place update_topm A/B (ablib/libcagra_inpl.so, hot-only build):
# C2 1M x 96 at M=896 p=16 forced on/off, then C4 10M x 96 at the 0.95 points
mkdir -p gpurun_out
L=$PWD/ablib/libcagra_inpl.so
for r in 1 2; do
  for f in 0 1; do
    CAGRA_LIB=$L CAGRA_SEARCH_INPLACE=$f timeout 300 python tools/sweep.py --grid "896,16,1,12,0,1" 2>&1 | tail -1 | sed "s/^/c2 inplace=$f /"
  done
done
for f in 0 1; do
  CAGRA_LIB=$L CAGRA_SEARCH_INPLACE=$f timeout 900 python tools/sweep.py --n 10000000 \
    --grid "3328,32,1,13,0,1;3328,16,1,13,0,1;3584,16,1,13,0,1;3072,16,1,13,0,1" 2>&1 | grep qps | sed "s/^/c4 inplace=$f /"
done
