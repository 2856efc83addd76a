mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_qd.py tests/test_gpu_scale.py tests/test_gpu_tso.py tests/test_cpp_dropin.py tests/test_gpu_multirank.py tests/test_gpu_native_islands.py -m gpu -q -x > gpurun_out/r2rng_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2rng_pytest.log
for c in cfg1 cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2rng_bench_$c.json 2> gpurun_out/r2rng_bench_$c.err
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1_r2rng.csv python tools/one_generation.py cfg1 64 5 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg1_r2rng.csv > gpurun_out/launches_cfg1_r2rng_summary.txt
