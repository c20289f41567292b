"""Stage-by-stage GPU smoke with flushed prints (debug aid)."""
import faulthandler
import sys
import time

faulthandler.dump_traceback_later(60, repeat=True)
sys.path.insert(0, ".")
import numpy as np

from oracle.bindings import load_oracle, make_params
from paper_2308_15136_b200 import capi, fodg

o = load_oracle()
t = time.time()


def log(*a):
    print(f"[{time.time() - t:7.2f}s]", *a, flush=True)


log("devices", capi.device_count())
data = o.uniform_dataset(300, 8, 1)
ds = fodg.Dataset.from_array(data)
ids, d = fodg.exact_topk_batch(ds, data[:5], 4)
log("topk ok", ids[0])
knn = fodg.exact_knn_graph(ds, 8)
oi, od = o.exact_knn_graph(data, 8)
log("knn equal", np.array_equal(knn.ids, oi))
c = fodg.count_detourable_routes(knn)
log("counts equal", np.array_equal(c, o.count_detourable_routes(oi, od)))
g = fodg.optimize(knn, 4)
log("opt equal", np.array_equal(g.ids, o.optimize(oi, od, 4)))
ix = fodg.Index(ds, g)
log("index ok")
q = o.uniform_dataset(4, 8, 2)
for exact in (True, False):
    for pol in (0, 1):
        r = ix.search(q, fodg.SearchParams(k=4, topm=16, width=2, hash_policy=fodg.HashPolicy(pol)),
                      fodg.EngineOptions(exact_distances=exact))
        ref = o.batch_search(g.ids, data, q, make_params(k=4, topm=16, width=2, hash_policy=pol))
        log("search exact", exact, "pol", pol, np.array_equal(r[0], ref[0]))
r = ix.search(q, fodg.SearchParams(k=4, topm=16), fodg.EngineOptions(mode=fodg.ExecutionMode(1)))
ref = o.batch_search(g.ids, data, q, make_params(k=4, topm=16), mode=1)
log("shared", np.array_equal(r[0], ref[0]))
