#!/bin/bash
# tools/build_cvariant.sh NAME "-DFLAG ..." : like build_variant.sh but recompiles only conv.cu
# (the other objects come from the main build in paper_1612_08825_b200/csrc/build)
set -e
cd "$(dirname "$0")/../paper_1612_08825_b200/csrc"
out=/tmp/ctcvar_$1; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr $2 -c conv.cu -o $out/conv.o
objs=$(ls build/*.o | grep -v conv.o)
mkdir -p ../../tools/variants
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o ../../tools/variants/$1.so $objs $out/conv.o
