mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_tso.py tests/test_gpu_evaluate.py tests/test_golden.py tests/test_gpu_qd.py -m gpu -q -x > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2o_pytest.log
