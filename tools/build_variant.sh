#!/bin/bash
# build_variant.sh name -Dflags... : a variant of the library under build_variants/ (A/B probes)
name=$1; shift
mkdir -p build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr "$@" -shared -o build_variants/libsgkkt_$name.so paper_2512_23804_b200/csrc/*.cu
