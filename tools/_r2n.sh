mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2n_pytest.log
for c in cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2n_bench_$c.json 2> gpurun_out/r2n_bench_$c.err
  TGB_NO_FUSED_KDAT=1 timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2n_bench_${c}_nofuse.json 2> gpurun_out/r2n_bench_${c}_nofuse.err
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r2n.csv python tools/one_generation.py cfg4 16384 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg4_r2n.csv > gpurun_out/launches_cfg4_r2n_summary.txt
