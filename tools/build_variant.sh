#!/bin/bash
# build a debug/experiment variant of the library: tools/build_variant.sh <name> [-DFLAG ...]
# -> build/var/lib<name>.so (load with LA_B200_LIB=build/var/lib<name>.so)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -I include "$@" -shared -cudart static -o build/var/lib$name.so paper_2405_17381_b200/csrc/*.cu
echo build/var/lib$name.so
