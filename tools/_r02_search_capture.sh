#!/bin/bash
# ncu --set full of the search kernel at the bench configuration (final
# round-2 kernel), summarised on the box; never a timing source
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 \
  -o /tmp/ncu/search python bench.py --steps 1 --warmup 3 --no-cpu --batch1 0 > gpurun_out/r02_search_full.log 2>&1
python tools/ncu_summary.py full /tmp/ncu/search.ncu-rep gpurun_out/r02_search_ncu.json --label r02 > /dev/null 2>&1
python tools/ncu_lines.py /tmp/ncu/search.ncu-rep 40 > gpurun_out/r02_search_stall_lines.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --batch1 20 \
  > gpurun_out/r02_launches_bench.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches.csv gpurun_out/r02_launches.txt > /dev/null 2>&1
