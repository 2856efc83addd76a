#!/bin/bash
# Bench lines, per-generation launch lists and ncu captures of the main
# kernels for cfg2 / cfg3 / cfg4 (run on the GPU box through gpurun; outputs
# in gpurun_out/, summarised into profiles/ by hand and tools/ncu_*.py).
#   usage: bash tools/profile_all.sh TAG
set -u
TAG=${1:-v}
OUT=gpurun_out
mkdir -p $OUT
for c in cfg1 cfg2 cfg3 cfg4; do
  python bench.py --config $c --steps 30 --warmup 5 > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err
done
for cb in "cfg2 4096" "cfg3 4096" "cfg4 16384"; do
  set -- $cb
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_${1}_$TAG.csv python tools/one_generation.py $1 $2 > /dev/null 2>&1
  python tools/launch_summary.py $OUT/launches_${1}_$TAG.csv > $OUT/launches_${1}_${TAG}_summary.txt
done
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k k_sweep --launch-skip 3 -c 1 -o $OUT/sweep_cfg2_$TAG python tools/step_timing.py cfg2 4096 > /dev/null 2>&1
$NCU -k k_sweep --launch-skip 3 -c 1 -o $OUT/sweep_cfg4_$TAG python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
$NCU -k k_sweep_masked --launch-skip 10 -c 1 -o $OUT/masked_cfg3_$TAG python tools/step_timing.py cfg3 4096 > /dev/null 2>&1
$NCU -k k_prep --launch-skip 3 -c 1 -o $OUT/prep_cfg2_$TAG python tools/step_timing.py cfg2 4096 > /dev/null 2>&1
$NCU -k k_prep --launch-skip 3 -c 1 -o $OUT/prep_cfg4_$TAG python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
ls -la $OUT
