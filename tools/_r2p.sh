mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_import.py -m gpu -q -x -s > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
for c in cfg4 cfg2; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2p_bench_$c.json 2> gpurun_out/r2p_bench_$c.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_prep_rows|k_finish" --launch-skip 8 -c 3 -o gpurun_out/prepfin_cfg4_r2p python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
