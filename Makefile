# Top-level build: the CUDA engine (sm_100a) and the oracle checkers.
#   make -j4        -> paper_0909_2000_b200/libalignplot_b200.so + oracle/
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $(EXTRA_NVFLAGS)
PKG := paper_0909_2000_b200
CSRC := $(PKG)/csrc
BUILD ?= build
LIB ?= $(PKG)/libalignplot_b200.so
OBJS := $(BUILD)/ap_capi.o $(BUILD)/ap_inst_l4.o $(BUILD)/ap_inst_l8.o $(BUILD)/ap_inst_l16.o $(BUILD)/ap_inst_l32.o $(BUILD)/ap_inst_r2.o $(BUILD)/ap_inst_r2hf.o $(BUILD)/ap_inst_ghf_a.o $(BUILD)/ap_inst_ghf_b.o $(BUILD)/ap_inst_ghf_c.o $(BUILD)/ap_inst_dual_a.o $(BUILD)/ap_inst_dual_b.o $(BUILD)/ap_inst_dual_c.o $(BUILD)/ap_inst_dual_d.o $(BUILD)/ap_inst_dual_r2.o
HDRS := $(CSRC)/ap_kernels.cuh $(CSRC)/ap_aux_kernels.cuh $(CSRC)/ap_wide_kernels.cuh $(CSRC)/ap_dual_kernels.cuh include/alignplot_b200.h

all: $(LIB) oracle

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

$(BUILD):
	mkdir -p $(BUILD) $(dir $(LIB))

# experiment builds: make variant V=name FLAGS="-DFOO" -> tools/exp/name/libalignplot_b200.so
# (load with AP_LIB_PATH=tools/exp/name/libalignplot_b200.so)
variant:
	mkdir -p tools/exp/$(V)
	$(MAKE) BUILD=/tmp/apbuild/$(V) LIB=tools/exp/$(V)/libalignplot_b200.so EXTRA_NVFLAGS="$(FLAGS)" \
	  tools/exp/$(V)/libalignplot_b200.so

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean variant

# C++ drop-in test (reference test cases against alignplot_shim.hpp); runs on a GPU box.
tests/cpp/test_shim: tests/cpp/test_shim.cpp $(CSRC)/alignplot_shim.hpp include/alignplot_b200.h $(LIB)
	g++ -std=c++20 -O2 -o $@ $< -L$(PKG) -lalignplot_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

all: tests/cpp/test_shim
