#!/bin/bash
# background GPU job: C3 (1M x 960) recall/QPS curve + C4 (10M x 96) bench line
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --n 1000000 --dim 960 --nq 1000 \
  --grid "896,16;2048,32;3072,48;4096,64;4096,128;512,1,0,0,0,1,1,64,2;1024,1,0,0,0,1,1,128,2;2048,1,0,0,0,1,1,128,2" \
  > gpurun_out/c3_curve.txt 2>&1
timeout 1800 python bench.py --points 10000000 --topm 3328 --width 32 --hash-bits 13 --build-once \
  --batch1 0 --no-opt-parity --cpu-topm 3328 --cpu-width 32 --steps 5 --warmup 3 \
  > gpurun_out/c4_bench.log 2>&1
