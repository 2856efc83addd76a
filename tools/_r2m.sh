mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ac.py -q > gpurun_out/r2m_ac.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_ac.log
for c in cfg1 ac118; do
  timeout 600 python bench.py --stage ac --config $c --steps 10 --warmup 3 > gpurun_out/r2m_ac_$c.json 2> gpurun_out/r2m_ac_$c.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prep_rows --launch-skip 4 -c 2 -o gpurun_out/preprows_cfg4_r2m python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ac_case --launch-skip 4 -c 1 -o gpurun_out/ac_case_ac118_r2m python bench.py --stage ac --config ac118 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
