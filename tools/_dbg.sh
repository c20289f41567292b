timeout 300 python tools/knn_check.py 0 > gpurun_out/knn_check5.log 2>&1
python tools/knn_prof.py 1000000 >> gpurun_out/knn_check5.log 2>&1
CAGRA_TC_DEBUG=3 python tools/knn_prof.py 1000000 >> gpurun_out/knn_check5.log 2>&1
python - >> gpurun_out/knn_check5.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, os
from paper_2308_15136_b200 import capi, fodg
for n, dim, k in [(100000, 96, 128), (200000, 37, 40), (70000, 128, 64)]:
    data = capi.uniform_dataset(n, dim, 5); ds = fodg.Dataset.from_array(data)
    os.environ['CAGRA_KNN_PATH'] = 'auto'; g = fodg.exact_knn_graph(ds, k); st = capi.knn_last_stats()
    os.environ['CAGRA_KNN_PATH'] = 'simt'; h = fodg.exact_knn_graph(ds, k)
    print(n, dim, k, st, 'rows identical', np.mean(np.all(g.ids == h.ids, 1)), 'dist bits', np.mean(g.dists.view(np.uint32) == h.dists.view(np.uint32)))
    q = capi.uniform_dataset(10000, dim, 6)
    os.environ['CAGRA_KNN_PATH'] = 'auto'; a = fodg.exact_topk_batch(ds, q, 10); st = capi.knn_last_stats()
    os.environ['CAGRA_KNN_PATH'] = 'simt'; b = fodg.exact_topk_batch(ds, q, 10)
    print('  gt', st, np.array_equal(a[0], b[0]), np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32)))
PY
