# Build libspa_b200.so for sm_100a (B200) only.  No CPU fallback exists.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC \
           -Xptxas -v --expt-relaxed-constexpr
SRC := paper_1106_0322_b200/csrc/spa_core.cu paper_1106_0322_b200/csrc/resample.cu paper_1106_0322_b200/csrc/mwg.cu \
       paper_1106_0322_b200/csrc/emmap.cu
HDR := $(wildcard paper_1106_0322_b200/csrc/*.cuh) include/spa_b200.h
LIB := paper_1106_0322_b200/libspa_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; false)

clean:
	rm -f $(LIB) build_ptxas.log
.PHONY: all clean
