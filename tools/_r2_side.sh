mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r2sd_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2sd_pytest.log
for c in cfg1 cfg4; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2sd_bench_$c.json 2> gpurun_out/r2sd_bench_$c.err
done
