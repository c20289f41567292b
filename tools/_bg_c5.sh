#!/bin/bash
# background GPU job: C5 (100M x 96) as 8 dataset shards of 12.5M on one B200
mkdir -p gpurun_out
free -g > gpurun_out/c5_free.txt
timeout 3000 python bench.py --points 100000000 --shard data --shards-per-rank 8 \
  --topm 3328 --width 32 --hash-bits 13 --steps 3 --warmup 3 --batch1 0 --no-cpu \
  > gpurun_out/c5_bench.log 2>&1
echo "rc=$?" >> gpurun_out/c5_bench.log
