#!/bin/bash
# K1 quick loop on the GPU box: timing (default + HV1), parity tests, launch list
mkdir -p gpurun_out
(timeout 200 python tools/knn_time.py; CAGRA_TC_HALVES=1 timeout 200 python tools/knn_time.py) > gpurun_out/kt.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "knn or ground_truth" > gpurun_out/knn_tests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/knn_launches3.csv python tools/knn_prof.py 1000000 96 128 > /dev/null 2>&1
(timeout 200 python tools/gt_time.py; CAGRA_TC_NOSPLIT=1 timeout 200 python tools/gt_time.py) > gpurun_out/gt.log 2>&1
