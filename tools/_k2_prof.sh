#!/bin/bash
# ncu --set full of the optimize kernels (K2 detour_reorder, K3, K4) of the
# 1M x 96 build, summarised on the box.  Never a timing source.
mkdir -p gpurun_out /tmp/ncu
for k in detour_reorder_kernel reverse_select_kernel merge_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 \
    -o /tmp/ncu/$k python tools/knn_time.py > gpurun_out/r02_${k}_full.log 2>&1
  python tools/ncu_summary.py full /tmp/ncu/$k.ncu-rep gpurun_out/r02_${k}_ncu.json --label r02 \
    > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/ncu/$k.ncu-rep 30 > gpurun_out/r02_${k}_stall_lines.txt 2>&1
done
