import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2308_15136_b200 import capi, fodg
data = capi.uniform_dataset(5000, 24, 1)
q = capi.uniform_dataset(4, 24, 2)
ds = fodg.Dataset.from_array(data)
g, _ = fodg.build_graph(ds, 16)
ix = fodg.Index(ds, g)
prm = fodg.SearchParams(k=10, topm=16, width=1, seed=11)
opt = fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=8, multi_cta=2)
for r in range(3):
    ids, d, c, st = ix.search(q, prm, opt)
print(ids[0], c)
