# Build of the B200-native CAGRA engine (sm_100a only).
#   make            -> paper_2308_15136_b200/lib/libcagra_b200.so (kernels + C ABI)
#                      paper_2308_15136_b200/lib/libfodg_b200.so  (C++ drop-in fodg:: API)
#                      oracle/liboracle.so, oracle/_ref/libfodg_ref.so (test checkers)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2308_15136_b200/csrc \
           -Wno-deprecated-gpu-targets
CXXFLAGS:= -O2 -std=c++20 -fPIC -ffp-contract=off -Iinclude -I/usr/local/cuda/include -Wall
PKG     := paper_2308_15136_b200
CU_SRC  := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJ  := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRC))
HOST_SRC:= $(wildcard $(PKG)/host/*.cpp)
HOST_OBJ:= $(patsubst $(PKG)/host/%.cpp,build/host_%.o,$(HOST_SRC))
LIB     := $(PKG)/lib/libcagra_b200.so
FODG    := $(PKG)/lib/libfodg_b200.so

CLI     := $(PKG)/lib/fodg

all: $(LIB) $(if $(HOST_SRC),$(FODG)) $(CLI) oracle refsuite tools dropintests

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/common.cuh $(PKG)/csrc/kernels.hpp $(PKG)/csrc/host_util.hpp include/cagra/capi.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(CU_OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $(CU_OBJ) -Xlinker -rpath -Xlinker /usr/local/cuda/lib64

build/host_%.o: $(PKG)/host/%.cpp $(wildcard include/fodg/*.hpp) include/cagra/capi.h
	@mkdir -p build
	g++ $(CXXFLAGS) -c $< -o $@

$(FODG): $(HOST_OBJ) $(LIB)
	g++ -shared -o $@ $(HOST_OBJ) -L$(PKG)/lib -lcagra_b200 -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,/usr/local/cuda/lib64

$(CLI): $(PKG)/cli/fodg_main.cpp $(FODG)
	g++ $(CXXFLAGS) -o $@ $< -L$(PKG)/lib -lfodg_b200 -lcagra_b200 -Wl,-rpath,'$$ORIGIN'

# The reference's own unit suites + acceptance binary, compiled unchanged from
# /root/reference against the drop-in (tests/compat/doctest.h stands in for the
# absent vendor/doctest).  Built artefacts only (tests/_refsuite, git-ignored);
# skipped when /root/reference is absent (the GPU box runs the prebuilt ones).
REFTESTS := /root/reference/proj/tests
SUITES   := test_core test_knn_build test_graph_opt test_search test_engine test_io test_graph_metrics
ifneq ($(wildcard $(REFTESTS)/test_core.cpp),)
refsuite: $(addprefix tests/_refsuite/,$(SUITES)) tests/_refsuite/acceptance
tests/_refsuite/%: $(REFTESTS)/%.cpp $(FODG) tests/compat/doctest.h $(wildcard include/fodg/*.hpp)
	@mkdir -p tests/_refsuite
	g++ -O2 -std=c++20 -ffp-contract=off -w -Iinclude -Itests/compat -I$(REFTESTS) -o $@ $< \
	    $(if $(filter acceptance,$*),,$(REFTESTS)/doctest_main.cpp) \
	    -L$(PKG)/lib -lfodg_b200 -lcagra_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -pthread
else
refsuite:
	@echo "refsuite: /root/reference absent; using prebuilt tests/_refsuite if any"
endif

# drop-in behaviour tests (C++ callers of fodg::, run by tests/test_dropin.py)
DROPIN_TESTS := tests/_dropin/test_dropin_cache
dropintests: $(DROPIN_TESTS)
tests/_dropin/%: tests/cpp/%.cpp $(FODG)
	@mkdir -p tests/_dropin
	g++ -O2 -std=c++20 -Iinclude -o $@ $< -L$(PKG)/lib -lfodg_b200 -lcagra_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib'

# measurement tools (C++ callers of the C ABI / the drop-in; not part of the product)
TOOLS := tools/cpp/b1_latency tools/cpp/dropin_bench
tools: $(TOOLS)
tools/cpp/%: tools/cpp/%.cpp $(FODG)
	g++ -O2 -std=c++20 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG)/lib -lfodg_b200 -lcagra_b200 \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -Wl,-rpath,/usr/local/cuda/lib64

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/lib

.PHONY: all oracle clean refsuite tools dropintests
