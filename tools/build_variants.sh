#!/bin/bash
# Build tuning variants of the library: build/variants/<name>/libdg2d_b200.so
# usage: tools/build_variants.sh name "NVCC defines" [name "defines"]...
set -e
cd "$(dirname "$0")/.."
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  out=build/variants/$name; rm -rf $out; mkdir -p $out/obj
  for p in 1 2 3 4 5; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $defs \
      -c paper_1601_07944_b200/csrc/device/kernels_p$p.cu -o $out/obj/kernels_p$p.o &
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $defs \
      -c paper_1601_07944_b200/csrc/device/solver.cu -o $out/obj/solver.o &
  wait
  for p in 1 2 3 4 5; do test -f $out/obj/kernels_p$p.o || { echo "variant $name failed"; exit 1; }; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libdg2d_b200.so $out/obj/*.o build/obj/basis.o build/obj/mesh.o build/obj/problems.o build/obj/capi_setup.o
  echo built $name
done
