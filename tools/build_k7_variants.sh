#!/bin/bash
# Dev: builds libgmcp_b200 variants of contact_eval.cu, one per argument
# NAME=DEFINES (e.g. mb5=-DK7_MINB=5) -> paper_2605_24339_b200/libgmcp_b200_NAME.so
set -e
cd "$(dirname "$0")/../paper_2605_24339_b200/csrc"
make -s
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for spec in "$@"; do
  name=${spec%%=*}; defs=${spec#*=}
  nvcc $F $defs -c contact_eval.cu -o build/contact_eval_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libgmcp_b200_$name.so build/capi.o build/contact_eval_$name.o build/exact.o build/plan.o build/sampler.o build/solver.o -lcudart
done
