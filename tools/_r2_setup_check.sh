mkdir -p gpurun_out
timeout 2000 python -m pytest tests/test_gpu_tso.py tests/test_gpu_scale.py tests/test_gpu_evaluate.py tests/test_gpu_ptdf.py -m gpu -q > gpurun_out/r2gj_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2gj_pytest.log
timeout 400 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2gj_bench_cfg4.json 2> gpurun_out/r2gj_bench_cfg4.err
