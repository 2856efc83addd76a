mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_tso.py -m gpu -q -x > gpurun_out/r2z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2z_pytest.log
for c in cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2z_bench_$c.json 2> gpurun_out/r2z_bench_$c.err
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r2z.csv python tools/one_generation.py cfg4 16384 5 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg4_r2z.csv > gpurun_out/launches_cfg4_r2z_summary.txt
