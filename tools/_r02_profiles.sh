#!/bin/bash
# round-2 evidence captures (one GPU): launch list of a bench run, ncu --set
# full of the search kernel (bench config), the K1 full pass and the batch-1
# team kernel; summarised ON the box (the .ncu-rep files stay in /tmp).
# Never a timing source.
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --batch1 20 \
  > gpurun_out/r02_launches_bench.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches.csv gpurun_out/r02_launches.txt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 \
  -o /tmp/ncu/search python bench.py --steps 1 --warmup 3 --no-cpu --batch1 0 > gpurun_out/r02_search_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_tc_kernel -s 1 -c 1 \
  -o /tmp/ncu/knn python tools/knn_prof.py 1000000 96 128 > gpurun_out/r02_knn_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:team_b1 -s 20 -c 1 \
  -o /tmp/ncu/b1 python tools/b1_device.py 10,96 > gpurun_out/r02_b1_full.log 2>&1
for r in search knn b1; do
  python tools/ncu_summary.py full /tmp/ncu/$r.ncu-rep gpurun_out/r02_${r}_ncu.json --label r02 \
    > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/ncu/$r.ncu-rep 40 > gpurun_out/r02_${r}_stall_lines.txt 2>&1
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/r02_${r}_raw.csv 2>/dev/null
done
ls -la /tmp/ncu gpurun_out/r02_* > gpurun_out/r02_ls.txt
