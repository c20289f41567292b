for v in new prev new prev; do
  if [ $v = new ]; then L=paper_2308_15136_b200/lib/libcagra_b200.so; else L=lib_variants/libcagra_prev.so; fi
  CAGRA_LIB=$L timeout 120 python tools/knn_prof.py 1000000 2>&1 | sed "s/^/$v /" | cut -c1-100 >> gpurun_out/knn_ab3.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -k "knn or gist or build or ground" -q 2>&1 | tail -1 >> gpurun_out/knn_ab3.log
