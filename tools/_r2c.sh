mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
for c in cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_$c.json 2> gpurun_out/r2c_bench_$c.err
done
TGB_NO_PHI_COLUMNS=1 timeout 400 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_cfg4_nophi.json 2> gpurun_out/r2c_bench_cfg4_nophi.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r2v2.csv python tools/one_generation.py cfg4 16384 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg4_r2v2.csv > gpurun_out/launches_cfg4_r2v2_summary.txt
