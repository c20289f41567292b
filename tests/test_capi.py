"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/cagra/capi.h declares, host helpers work, and compute calls
fail loudly (CAGRA_ERR_CUDA) instead of falling back to the CPU when no
device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2308_15136_b200 import capi, fodg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cagra", "capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cagra_[a-z0-9_]+)\s*\(", src)))


def test_header_declarations_match_binding_list():
    assert declared_symbols() == sorted(capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_fodg_shim_exports_reference_api():
    path = os.path.join(ROOT, "paper_2308_15136_b200", "lib", "libfodg_b200.so")
    if not os.path.exists(path):
        pytest.skip("C++ drop-in shim not built")
    out = os.popen(f"nm -DC {path}").read()
    for sym in ["fodg::batch_search", "fodg::optimize", "fodg::exact_knn_graph",
                "fodg::search_one", "fodg::choose_mode", "fodg::run_benchmark",
                "fodg::exact_topk", "fodg::count_detourable_routes", "fodg::merge_graphs",
                "fodg::build_reverse_graph", "fodg::reorder_and_prune", "fodg::update_topm"]:
        assert sym in out, sym


def test_host_helpers():
    assert capi.mix_seed(0) == 0xE220A8397B1DCDAF
    a = capi.uniform_dataset(4, 3, 1)
    assert a.dtype == np.float32 and a.shape == (4, 3) and (a >= 0).all() and (a < 1).all()
    assert "sm_100a" in capi.lib().cagra_version().decode()


def test_struct_layouts_match_header():
    assert C.sizeof(capi.SearchParamsC) == 40
    assert C.sizeof(capi.EngineOptsC) == 40
    assert C.sizeof(capi.SearchStatsC) == 24 == capi.STATS_DTYPE.itemsize
    p = C.create_string_buffer(40)
    capi.lib().cagra_search_params_default(p)
    sp = capi.SearchParamsC.from_buffer_copy(p.raw)
    assert (sp.k, sp.topm, sp.width, sp.hash_bits, sp.reset_interval) == (10, 64, 1, 11, 1)


def test_compute_fails_loudly_without_device():
    if capi.device_count() > 0:
        pytest.skip("a CUDA device is present")
    ds = fodg.Dataset(2, np.arange(8, dtype=np.float32))
    with pytest.raises(capi.CudaError):
        fodg.exact_knn_graph(ds, 1)
    with pytest.raises(capi.CudaError):
        fodg.Index(ds, fodg.Graph(4, 1, np.array([[1], [0], [3], [2]], np.uint32)))


def test_argument_validation_precedes_device_use():
    # UsageError is raised in the reference's order even without a device
    ds = fodg.Dataset(1, [0, 1, 3, 7])
    with pytest.raises(capi.UsageError):
        fodg.exact_knn_graph(ds, 4)
    g = fodg.KnnGraph(2, 1, np.array([[1], [0]], np.uint32), np.ones((2, 1), np.float32))
    with pytest.raises(capi.UsageError):
        fodg.optimize(g, 2)


def test_graph_metrics_host_side():
    # graph_metrics.hpp: empty graph needs no device; the report is the
    # reference's key=value lines; compute needs the device (no CPU fallback)
    empty = fodg.Graph(0, 4, np.zeros((0, 4), np.uint32))
    r = fodg.measure_graph(empty)
    assert (r.strong_cc, r.avg_2hop, r.max_2hop) == (0, 0.0, 20)
    assert fodg.GraphQualityReport(3, 2, 1, 1.5, 6).report() == (
        "num_nodes=3\ndegree=2\nstrong_cc=1\navg_2hop=1.5\nmax_2hop=6\n")
    if capi.device_count() == 0:
        with pytest.raises(capi.CudaError):
            fodg.measure_graph(fodg.Graph(2, 1, np.array([[1], [0]], np.uint32)))
