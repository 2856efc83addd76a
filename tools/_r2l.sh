mkdir -p gpurun_out
for c in cfg1 ac118; do
  timeout 600 python bench.py --stage ac --config $c --steps 10 --warmup 3 > gpurun_out/r2l_ac_$c.json 2> gpurun_out/r2l_ac_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_ac_launches.csv python bench.py --stage ac --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ac_case --launch-skip 4 -c 1 -o gpurun_out/ac_case_cfg1_r2l python bench.py --stage ac --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
