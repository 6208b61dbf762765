#!/bin/bash
# Dev: builds libgmcp_b200 variants with different K7 launch bounds (K7_MINB).
set -e
cd "$(dirname "$0")/../paper_2605_24339_b200/csrc"
make -s
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for mb in "$@"; do
  nvcc $F -DK7_MINB=$mb -c contact_eval.cu -o build/contact_eval_mb$mb.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libgmcp_b200_mb$mb.so build/capi.o build/contact_eval_mb$mb.o build/exact.o build/sampler.o build/solver.o -lcudart
done
