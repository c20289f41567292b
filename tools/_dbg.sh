timeout 300 python tools/knn_check.py 0 > gpurun_out/knn_check8.log 2>&1
python tools/knn_prof.py 1000000 >> gpurun_out/knn_check8.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -k "knn or gist or build" -q >> gpurun_out/knn_check8.log 2>&1
