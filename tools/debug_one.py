import sys; sys.path.insert(0, ".")
import numpy as np
from oracle.bindings import load_oracle
from paper_2308_15136_b200 import fodg
o = load_oracle()
data = o.uniform_dataset(300, 8, 1); ds = fodg.Dataset.from_array(data)
g = fodg.optimize(fodg.exact_knn_graph(ds, 8), 4)
ix = fodg.Index(ds, g); q = o.uniform_dataset(1, 8, 2)
r = ix.search(q, fodg.SearchParams(k=4, topm=16, width=2), fodg.EngineOptions(exact_distances=False, team_size=8))
print("done", r[0], flush=True)
