# Builds the sm_100a shared library in-tree (it travels to the GPU box).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
SRC := $(wildcard paper_2512_23804_b200/csrc/*.cu)
LIB := paper_2512_23804_b200/libsgkkt_b200.so

all: $(LIB)

$(LIB): $(SRC) paper_2512_23804_b200/csrc/sgk_common.cuh include/sgkkt_b200.h
	$(NVCC) $(ARCH) $(NVFLAGS) -shared -o $@ $(SRC)

# trace build of the wide triangular solve (tools/triw_trace.py)
trace: $(SRC)
	mkdir -p build_variants && $(NVCC) $(ARCH) $(NVFLAGS) -DSGK_TRIW_TRACE -shared -o build_variants/libsgkkt_triwtrace.so $(SRC)

# phase-trace build of the warp-specialised matvec kernel (tools/s9_trace.py)
s9trace: $(SRC)
	mkdir -p build_variants && $(NVCC) $(ARCH) $(NVFLAGS) -DSGK_S9_TRACE -shared -o build_variants/libsgkkt_s9trace.so $(SRC)

ptxas:
	$(NVCC) $(ARCH) $(NVFLAGS) -Xptxas -v -c -o /tmp/sgk_probe.o paper_2512_23804_b200/csrc/galerkin.cu

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas trace s9trace
