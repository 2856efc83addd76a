# AC stage launch list (per-kernel device time) for cfg1: $1 = tag
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$1_ac_launches_cfg1.csv python bench.py --stage ac --config cfg1 --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/$1_ac_ncu_cfg1.log 2>&1
