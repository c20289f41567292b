#!/bin/bash
# round-2 re-entry: guard-zone tests, random-gather ceiling, eval-prefetch A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_guard_zones.py -x -q > gpurun_out/guard.log 2>&1; tail -3 gpurun_out/guard.log
timeout 300 tools/cpp/gather_peak > gpurun_out/gather_peak.txt 2>&1
AB_LIBS="pf1 pf2" AB_REPS=3 timeout 1500 bash tools/_ab.sh > gpurun_out/pf_ab.txt 2>&1
