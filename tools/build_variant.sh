#!/bin/bash
# Build an A/B variant of libprefill_sm100.so with extra nvcc -D flags on gemm.cu / attention.cu / mlp.cu:
#   tools/build_variant.sh NAME -DPF_RING_STAGES=5 -DPF_RB_DEPTH=2   -> variants/NAME/libprefill_sm100.so
# Use it with PF_LIB_PATH=variants/NAME/libprefill_sm100.so (variants/ is git-ignored, but travels).
set -e
cd "$(dirname "$0")/../paper_2510_22101_b200/csrc"
name=$1; shift
out=../../variants/$name; mkdir -p $out/obj
make -s
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
for f in gemm attention mlp; do nvcc $FL "$@" -c $f.cu -o $out/obj/$f.o; done
nvcc $ARCH -shared -o $out/libprefill_sm100.so $out/obj/gemm.o $out/obj/attention.o $out/obj/mlp.o build/capi.o build/elementwise.o \
  build/host_ingest.o -lcudart_static -ldl -lrt -lpthread
echo "built $out/libprefill_sm100.so"
