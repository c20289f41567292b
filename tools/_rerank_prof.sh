#!/bin/bash
# ncu --set full of the K1 append-mode re-rank (1M x 96 k=128), summarised on the box
mkdir -p gpurun_out /tmp/ncu
k=tc_rerank_append_kernel
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 \
  -o /tmp/ncu/$k python tools/knn_time.py > gpurun_out/r02_${k}_full.log 2>&1
python tools/ncu_summary.py full /tmp/ncu/$k.ncu-rep gpurun_out/r02_${k}_ncu.json --label r02 > /dev/null 2>&1
python tools/ncu_lines.py /tmp/ncu/$k.ncu-rep 30 > gpurun_out/r02_${k}_stall_lines.txt 2>&1
