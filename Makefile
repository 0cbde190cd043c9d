# Top-level build: the CUDA engine (sm_100a) and the oracle checkers.
#   make            -> paper_0909_2000_b200/libalignplot_b200.so + oracle/
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
PKG := paper_0909_2000_b200
LIB := $(PKG)/libalignplot_b200.so
SRCS := $(PKG)/csrc/ap_capi.cu
HDRS := $(PKG)/csrc/ap_kernels.cuh include/alignplot_b200.h

all: $(LIB) oracle

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> build/ptxas.log || (cat build/ptxas.log; false)

oracle:
	$(MAKE) -C oracle

$(shell mkdir -p build)

clean:
	rm -f $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
