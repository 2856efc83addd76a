# ncu --set full of the AC case kernel at cfg1: $1 = tag
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ac_case --launch-skip 4 -c 1 \
  -o gpurun_out/ac_case_cfg1_$1 python bench.py --stage ac --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$1_acfull.log 2>&1
