#!/bin/bash
# tools/build_variant.sh NAME "-DFLAG ..." : build the library with extra nvcc flags into tools/variants/NAME.so
set -e
cd "$(dirname "$0")/../paper_1612_08825_b200/csrc"
out=/tmp/ctvar_$1; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in common conv ttc moments tma host_stream synth gradient ingest; do
  if [ "$f" = moments ] || [ "$f" = ttc ] || [ "$f" = conv ] || [ ! -f $out/$f.o ]; then
    /usr/local/cuda/bin/nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr $2 -c $f.cu -o $out/$f.o &
  fi
done
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o ../../tools/variants/$1.so $out/*.o
