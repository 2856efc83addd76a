mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2h_pytest.log
for c in cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_$c.json 2> gpurun_out/r2h_bench_$c.err
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r2v6.csv python tools/one_generation.py cfg4 16384 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg4_r2v6.csv > gpurun_out/launches_cfg4_r2v6_summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prep_rows --launch-skip 6 -c 1 -o gpurun_out/preprows_cfg4_r2v6 python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_chunked --launch-skip 2 -c 1 -o gpurun_out/chunked_cfg4_r2v6 python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
