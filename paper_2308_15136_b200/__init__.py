"""B200-native CAGRA engine: sm_100a kernels behind the reference's fodg:: API.

    from paper_2308_15136_b200 import fodg
    g, info = fodg.build_graph(ds, d=64)          # exact kNN + rank optimize, on device
    res = fodg.batch_search(g, ds, queries, fodg.SearchParams(topm=256, width=4), opts)

The compute path is libcagra_b200.so (built by `make`); see include/cagra/capi.h.
"""
__version__ = "0.1.0"
