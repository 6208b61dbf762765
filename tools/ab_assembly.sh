#!/bin/bash
# A/B helper (GPU box): contact/full-size GPU tests, then the assembly bench N times.
#   bash tools/ab_assembly.sh [N]
python -m pytest tests -m gpu -x -q -k "contact or fullsize or gather or batch or dropin" 2>&1 | tail -1
for i in $(seq ${1:-2}); do
  python bench.py --no-cpu-baseline --no-newton --no-batched --steps 50 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pass_us %.1f  k7_us %.1f  value %.4g  e2e %.4g' % (d['ms_per_step']*1e3, d['roofline']['ms']*1e3, d['value'], d['e2e']['value']))"
done
