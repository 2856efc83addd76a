mkdir -p gpurun_out
for c in cfg4 cfg2 cfg1 cfg3; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2s_bench_$c.json 2> gpurun_out/r2s_bench_$c.err
done
for c in cfg1 cfg4; do
  B=$(python -c "from bench import CONFIGS; print(CONFIGS['$c']['batch'])")
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_r2s.csv python tools/one_generation.py $c $B 5 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_${c}_r2s.csv > gpurun_out/launches_${c}_r2s_summary.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o gpurun_out/chunked_cfg4_r2s python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
