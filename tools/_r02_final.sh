#!/bin/bash
# round-2 closing evidence on one GPU: full GPU suite, bench (our arm and the
# reference arm), then the launch list and ncu --set full summaries
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final_gputests.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 2400 bash tools/_r02_profiles.sh
