# Top-level build: the CUDA engine (sm_100a) and the oracle checkers.
#   make -j4        -> paper_0909_2000_b200/libalignplot_b200.so + oracle/
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $(EXTRA_NVFLAGS)
PKG := paper_0909_2000_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libalignplot_b200.so
OBJS := build/ap_capi.o build/ap_inst_l8.o build/ap_inst_l16.o build/ap_inst_l32.o build/ap_inst_r2.o
HDRS := $(CSRC)/ap_kernels.cuh $(CSRC)/ap_aux_kernels.cuh include/alignplot_b200.h

all: $(LIB) oracle

build/%.o: $(CSRC)/%.cu $(HDRS) | build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

build:
	mkdir -p build

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

# C++ drop-in test (reference test cases against alignplot_shim.hpp); runs on a GPU box.
tests/cpp/test_shim: tests/cpp/test_shim.cpp $(CSRC)/alignplot_shim.hpp include/alignplot_b200.h $(LIB)
	g++ -std=c++20 -O2 -o $@ $< -L$(PKG) -lalignplot_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

all: tests/cpp/test_shim
