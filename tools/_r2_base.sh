mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
lscpu > gpurun_out/lscpu.txt; free -g > gpurun_out/free.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2base.log 2>&1; tail -2 gpurun_out/gputests_r2base.log
timeout 900 python bench.py > gpurun_out/bench_r2base.json 2> gpurun_out/bench_r2base.err
