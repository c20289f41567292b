timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c1_parity.py -x -q -k "knn or ground_truth or c1 or build_graph" 2>&1 | tail -2
bash tools/_knn_ab.sh rrold
