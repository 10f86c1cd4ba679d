# Builds the sm_100a shared library in-tree (it travels to the GPU box).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
SRC := $(wildcard paper_2512_23804_b200/csrc/*.cu)
LIB := paper_2512_23804_b200/libsgkkt_b200.so

all: $(LIB)

$(LIB): $(SRC) paper_2512_23804_b200/csrc/sgk_common.cuh include/sgkkt_b200.h
	$(NVCC) $(ARCH) $(NVFLAGS) -shared -o $@ $(SRC) -lcublas -Xlinker -rpath,/usr/local/cuda/lib64

ptxas:
	$(NVCC) $(ARCH) $(NVFLAGS) -Xptxas -v -c -o /tmp/sgk_probe.o paper_2512_23804_b200/csrc/galerkin.cu

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas
