#!/bin/bash
# launch times of the exact (line-search) kernels inside three C3 Newton iterations (GPU box)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_energy|k_step_filter|k_cap_active|k_true_resid|k_pair_jacobi" -c 60 --csv \
    --log-file gpurun_out/exact_launches.csv python tools/newton_c3.py 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/exact_launches.csv')))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
t = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        t[r[ki].split('(')[0][-40:]].append(float(r[vi].replace(',', '')) / 1e3)
for k, v in t.items():
    print('%-40s n=%2d mean %7.1f us' % (k, len(v), sum(v) / len(v)))
PY
