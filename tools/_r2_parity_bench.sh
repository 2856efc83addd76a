mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_tso.py tests/test_gpu_evaluate.py tests/test_gpu_capacity.py tests/test_golden.py tests/test_gpu_timesteps.py -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2u_pytest.log
for c in cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2u_bench_$c.json 2> gpurun_out/r2u_bench_$c.err
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r2u.csv python tools/one_generation.py cfg4 16384 5 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg4_r2u.csv > gpurun_out/launches_cfg4_r2u_summary.txt
