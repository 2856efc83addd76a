mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2j_pytest.log
for c in cfg4 cfg2 cfg1 cfg3; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2j_bench_$c.json 2> gpurun_out/r2j_bench_$c.err
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2j_bench_ref.json 2> gpurun_out/r2j_bench_ref.err
bash tools/profile_r2.sh r2j cfg4 cfg2 cfg1
