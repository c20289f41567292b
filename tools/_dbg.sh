for m in 0 1 2; do CAGRA_TC_DEBUG=$m python tools/knn_prof.py 1000000 2>&1 | tail -1 | sed "s/^/dbg=$m /"; done > gpurun_out/knn_dbg.log 2>&1
