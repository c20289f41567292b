# Build of the B200-native CAGRA engine (sm_100a only).
#   make            -> paper_2308_15136_b200/lib/libcagra_b200.so (kernels + C ABI)
#                      paper_2308_15136_b200/lib/libfodg_b200.so  (C++ drop-in fodg:: API)
#                      oracle/liboracle.so, oracle/_ref/libfodg_ref.so (test checkers)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2308_15136_b200/csrc \
           -Wno-deprecated-gpu-targets
CXXFLAGS:= -O2 -std=c++20 -fPIC -Iinclude -Wall
PKG     := paper_2308_15136_b200
CU_SRC  := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJ  := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRC))
HOST_SRC:= $(wildcard $(PKG)/host/*.cpp)
HOST_OBJ:= $(patsubst $(PKG)/host/%.cpp,build/host_%.o,$(HOST_SRC))
LIB     := $(PKG)/lib/libcagra_b200.so
FODG    := $(PKG)/lib/libfodg_b200.so

all: $(LIB) $(if $(HOST_SRC),$(FODG)) oracle

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/common.cuh $(PKG)/csrc/kernels.hpp include/cagra/capi.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(CU_OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $(CU_OBJ) -Xlinker -rpath -Xlinker /usr/local/cuda/lib64

build/host_%.o: $(PKG)/host/%.cpp $(wildcard include/fodg/*.hpp) include/cagra/capi.h
	@mkdir -p build
	g++ $(CXXFLAGS) -c $< -o $@

$(FODG): $(HOST_OBJ) $(LIB)
	g++ -shared -o $@ $(HOST_OBJ) -L$(PKG)/lib -lcagra_b200 -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/lib

.PHONY: all oracle clean
