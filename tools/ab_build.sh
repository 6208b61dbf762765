#!/bin/bash
# Same-box A/B of compile-time variants (GPU box, repo root):
#   bash tools/ab_build.sh "-DK7_ASYNC_META=0" "-DK7_ASYNC_META=1"
# rebuilds the library with each flag set and runs the assembly bench twice.
for f in "$@"; do
  touch paper_2605_24339_b200/csrc/assembly.cuh
  make -s -C paper_2605_24339_b200/csrc NVCC="nvcc $f" >/dev/null 2>&1 || { echo "build failed: $f"; continue; }
  for i in 1 2; do
    python bench.py --no-cpu-baseline --no-newton --no-batched --steps 50 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f pass_us %.1f  k7_us %.1f' % (d['ms_per_step']*1e3, d['roofline']['ms']*1e3))"
  done
done
