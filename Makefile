# Builds libparsmc_b200.so in-tree for sm_100a (B200).  -fmad=false keeps the
# reference's un-fused numpy evaluation order; wanted FMAs are explicit fma().
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS = -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v \
          --expt-relaxed-constexpr
SRC = paper_1212_1639_b200/csrc/engine.cu
HDR = $(wildcard paper_1212_1639_b200/csrc/*.cuh) $(wildcard paper_1212_1639_b200/csrc/*.inc) include/parsmc_b200.h
LIB = paper_1212_1639_b200/libparsmc_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

clean:
	rm -f $(LIB) build_ptxas.log

.PHONY: all clean
