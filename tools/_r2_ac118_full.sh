# AC checks + ncu --set full of the AC case kernel at ac118: $1 = tag
bash tools/_r2_ac_check.sh
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_ac_case --launch-skip 3 -c 1 \
  -o gpurun_out/ac_case_ac118_$1 python bench.py --stage ac --config ac118 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$1_ac118full.log 2>&1
