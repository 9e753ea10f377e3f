# Builds the B200-native DDPMA library (sm_100a) in-tree:
#   paper_2006_14602_b200/libddpma.so
# and the CPU oracle's C helpers (oracle/_build).  `python -c "import
# __graft_entry__ as g; g.build()"` runs this.

NVCC ?= nvcc
CXX ?= g++
SRC := paper_2006_14602_b200/csrc
OUT := paper_2006_14602_b200/libddpma.so
ARCH := -gencode arch=compute_100a,code=sm_100a
# -fmad=false / -ffp-contract=off: no multiply-add contraction, so every
# expression rounds exactly like the reference's numpy/Python arithmetic.
# DDPMA_MINB2=3: the 2D window kernels at 80 registers, 3 CTAs per SM (measured on B200:
# +11 % over 64 registers x 4 CTAs, +11 % over 128 registers x 2 CTAs; profiles/r2_variants.md)
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -v -DDDPMA_MINB2=3 \
           -Xcompiler -fPIC,-ffp-contract=off,-O2 -Iinclude
CXXFLAGS := -O2 -fPIC -std=c++17 -ffp-contract=off -Iinclude

OBJ := build/decomp.o build/plan.o build/kernels.o build/persist.o build/fileio.o

all: $(OUT)

build:
	mkdir -p build

build/decomp.o: $(SRC)/decomp.cpp $(SRC)/ddpma_internal.h include/ddpma.h | build
	$(CXX) $(CXXFLAGS) -c $< -o $@

build/fileio.o: $(SRC)/fileio.cpp include/ddpma.h | build
	$(CXX) $(CXXFLAGS) -pthread -c $< -o $@

build/plan.o: $(SRC)/plan.cu $(SRC)/ddpma_internal.h include/ddpma.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/plan.ptxas.log || (cat build/plan.ptxas.log; false)

build/kernels.o: $(SRC)/kernels.cu $(SRC)/ddpma_internal.h $(SRC)/stencil.cuh $(SRC)/fastlog.cuh $(SRC)/logtable.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/kernels.ptxas.log || (cat build/kernels.ptxas.log; false)

build/persist.o: $(SRC)/persist.cu $(SRC)/crpow.cuh $(SRC)/ddpma_internal.h $(SRC)/stencil.cuh $(SRC)/fastlog.cuh $(SRC)/logtable.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/persist.ptxas.log || (cat build/persist.ptxas.log; false)

$(OUT): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -Xcompiler -pthread

clean:
	rm -rf build $(OUT)

.PHONY: all clean
