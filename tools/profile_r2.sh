#!/bin/bash
# Round-2 evidence run (GPU box, via gpurun): launch lists of one generation
# per config and ncu --set full captures of the top kernels.
#   usage: bash tools/profile_r2.sh TAG [configs...]
set -u
TAG=${1:-v}; shift || true
CFGS=${@:-cfg1 cfg2 cfg4}
OUT=gpurun_out
mkdir -p $OUT
for c in $CFGS; do
  B=$(python -c "from bench import CONFIGS; print(CONFIGS['$c']['batch'])")
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_${c}_$TAG.csv python tools/one_generation.py $c $B > /dev/null 2>&1
  python tools/launch_summary.py $OUT/launches_${c}_$TAG.csv > $OUT/launches_${c}_${TAG}_summary.txt
done
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o $OUT/chunked_cfg4_$TAG python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
$NCU -k regex:k_prep --launch-skip 3 -c 1 -o $OUT/prep_cfg4_$TAG python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
$NCU -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o $OUT/chunked_cfg2_$TAG python tools/step_timing.py cfg2 4096 > /dev/null 2>&1
ls -la $OUT
