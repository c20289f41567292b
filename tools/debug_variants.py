"""Run each search-kernel variant in its own process with a timeout (debug aid)."""
import subprocess
import sys

code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
from oracle.bindings import load_oracle, make_params
from paper_2308_15136_b200 import fodg
o = load_oracle()
dim = int(sys.argv[1]); team = int(sys.argv[2]); mode = int(sys.argv[3]); nq = int(sys.argv[4])
data = o.uniform_dataset(300, dim, 1); ds = fodg.Dataset.from_array(data)
knn = fodg.exact_knn_graph(ds, 8); g = fodg.optimize(knn, 4)
ix = fodg.Index(ds, g); q = o.uniform_dataset(nq, dim, 2)
r = ix.search(q, fodg.SearchParams(k=4, topm=16, width=2), fodg.EngineOptions(
    mode=fodg.ExecutionMode(mode), exact_distances=False, team_size=team))
ref = o.batch_search(g.ids, data, q, make_params(k=4, topm=16, width=2), mode=mode)
print("ok", np.mean(r[0] == ref[0]), flush=True)
'''
cases = [("8", "0", "0", "1"), ("8", "32", "0", "1"), ("8", "8", "0", "1"), ("8", "16", "0", "1"),
         ("8", "4", "0", "1"), ("96", "0", "0", "4"), ("8", "0", "1", "2"), ("8", "0", "0", "64")]
for args in cases:
    try:
        p = subprocess.run([sys.executable, "-c", code, *args], capture_output=True, text=True,
                           timeout=25)
        print(args, p.stdout.strip()[-200:], p.stderr.strip()[-300:], flush=True)
    except subprocess.TimeoutExpired:
        print(args, "TIMEOUT", flush=True)
