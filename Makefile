# blinkline_b200 build: sm_100a only.
#
#   make            -> paper_2006_00816_b200/libblinkline_b200.so   (CUDA kernels + C-ABI)
#                      paper_2006_00816_b200/libblinkline_gpu.so    (C++ drop-in API over the C-ABI)
#                      oracle/liboracle.so                          (test-only C oracle)
#   make ref        -> oracle/_ref/libblinkline_ref.so              (reference, needs /root/reference)
#
# Exactness: the TUs that must reproduce the reference bit-for-bit are compiled with
# --fmad=false (no FMA contraction); only bl_classify.cu (the fp32 screen) and the host
# code keep contraction.

NVCC     ?= nvcc
CXX      ?= g++
PKG      := paper_2006_00816_b200
CSRC     := $(PKG)/csrc
BUILD    := build
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
EXACT    := --fmad=false
LIB      := $(PKG)/libblinkline_b200.so
CPPLIB   := $(PKG)/libblinkline_gpu.so

EXACT_CU := bl_pyramid bl_hog bl_exact bl_ert
FAST_CU  := bl_classify bl_screen_tc bl_capi
JSON_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
HOST_CPP := bl_io bl_run bl_multi
OBJS     := $(addprefix $(BUILD)/,$(addsuffix .o,$(EXACT_CU) $(FAST_CU) $(HOST_CPP)))
HDRS     := $(CSRC)/bl_internal.cuh include/blinkline_b200.h

all: $(LIB) $(CPPLIB) tests/cpp/test_dropin oracle

$(BUILD):
	@mkdir -p $(BUILD)

$(addprefix $(BUILD)/,$(addsuffix .o,$(EXACT_CU))): $(BUILD)/%.o: $(CSRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) $(EXACT) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(addprefix $(BUILD)/,$(addsuffix .o,$(FAST_CU))): $(BUILD)/%.o: $(CSRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(BUILD)/bl_io.o: $(CSRC)/bl_io.cpp include/blinkline_b200.h | $(BUILD)
	$(CXX) -std=c++17 -O2 -fPIC -I$(JSON_DIR) -c $< -o $@

$(BUILD)/bl_run.o: $(CSRC)/bl_run.cpp include/blinkline_b200.h | $(BUILD)
	$(CXX) -std=c++17 -O2 -fPIC -c $< -o $@

$(BUILD)/bl_multi.o: $(CSRC)/bl_multi.cpp include/blinkline_b200.h | $(BUILD)
	$(CXX) -std=c++17 -O2 -fPIC -Wall -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fPIC -lcudart_static -lrt -lpthread -ldl

$(CPPLIB): $(PKG)/cpp/blinkline_gpu.cpp $(PKG)/cpp/blinkline_gpu.hpp include/blinkline_b200.h $(LIB)
	$(CXX) -std=c++20 -O2 -fPIC -shared -I$(PKG)/cpp -Iinclude -o $@ $(PKG)/cpp/blinkline_gpu.cpp \
	  -L$(PKG) -lblinkline_b200 -Wl,-rpath,'$$ORIGIN'

tests/cpp/test_dropin: tests/cpp/test_dropin.cpp $(CPPLIB)
	$(CXX) -std=c++20 -O2 -pthread -I$(PKG)/cpp -o $@ $< -L$(PKG) -lblinkline_gpu -lblinkline_b200 \
	  -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

oracle:
	$(MAKE) -s -C oracle

ref:
	$(MAKE) -s -C oracle ref

clean:
	rm -rf $(BUILD) $(LIB) $(CPPLIB) tests/cpp/test_dropin

.PHONY: all oracle ref clean
