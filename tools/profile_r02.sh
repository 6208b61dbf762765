#!/bin/bash
# ncu captures summarised in profiles/r02/ (run on the GPU box from the repo root):
#   bash tools/profile_r02.sh   -> gpurun_out/prof_r02/
set -e
O=gpurun_out/prof_r02
mkdir -p $O
# launch list of the default assembly bench (cold, serialised: shares only)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --no-cpu-baseline --no-newton --no-batched --steps 3 --warmup 3 \
    > $O/launches.log 2>&1
# K7 / K8 full sets on the C3 assembly pass
ncu --set full --clock-control none --import-source on -k regex:k_run_partials -s 2 -c 1 -o $O/k7 \
    python tools/k7_time.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather -s 2 -c 1 -o $O/k8 \
    python tools/k7_time.py > /dev/null 2>&1
# the PCG kernels inside the C3 Newton solve (steady iteration: skip the first solves)
ncu --set full --clock-control none --import-source on -k regex:k_spmv_cg -s 600 -c 1 -o $O/spmv \
    python tools/newton_c3.py 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_update_agg -s 600 -c 1 -o $O/update_agg \
    python tools/newton_c3.py 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_coarse_prolong -s 600 -c 1 -o $O/coarse_prolong \
    python tools/newton_c3.py 3 > /dev/null 2>&1
# per-launch durations of one steady PCG stretch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_pupdate|k_spmv_cg|k_update_agg|k_coarse_prolong" -s 2400 -c 80 --csv --log-file $O/pcg_launches.csv \
    python tools/newton_c3.py 3 > /dev/null 2>&1
# the cooperative blocked Gauss-Jordan coarse inverse (704 coarse dofs, one launch) and the p-update
ncu --set full --clock-control none --import-source on -k regex:k_gj_persistent -s 1 -c 1 -o $O/gj_persistent \
    python tools/newton_c3.py 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pupdate -s 600 -c 1 -o $O/pupdate \
    python tools/newton_c3.py 3 > /dev/null 2>&1
# the per-scene CTA PCG (C5, two-level): shared-memory variant (default) and the global one
ncu --set full --clock-control none -k regex:k_pcg_scene -s 4 -c 1 -o $O/pcg_scene_sm python tools/c5_newton.py 1024 4 \
    > /dev/null 2>&1
GMCP_SCENE_SMEM=0 ncu --set full --clock-control none -k regex:k_pcg_scene -s 4 -c 1 -o $O/pcg_scene \
    python tools/c5_newton.py 1024 4 > /dev/null 2>&1
# the C3 rebuild's sampler kernels (warm rebuilds)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_sample|k_face|k_query|k_features|k_point_owner|k_tasks" -c 40 --csv --log-file $O/rebuild_launches.csv \
    python tools/rebuild_c3.py > /dev/null 2>&1
ls -la $O
