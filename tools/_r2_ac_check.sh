mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ac.py tests/test_cpp_dropin.py -m gpu -q -x > gpurun_out/r2ac_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ac_pytest.log
for c in cfg1 ac118; do
  timeout 600 python bench.py --stage ac --config $c --steps 10 --warmup 3 > gpurun_out/r2ac_bench_$c.json 2> gpurun_out/r2ac_bench_$c.err
done
