#!/bin/bash
# tools/build_mvariant.sh NAME "-DFLAG ..." : like build_variant.sh but recompiles only moments.cu
# (the other objects come from the main build in paper_1612_08825_b200/csrc/build)
set -e
cd "$(dirname "$0")/../paper_1612_08825_b200/csrc"
out=/tmp/ctmvar_$1; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr $2 -c moments.cu -o $out/moments.o
objs=$(ls build/*.o | grep -v moments.o)
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o ../../tools/variants/$1.so $objs $out/moments.o
