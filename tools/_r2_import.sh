mkdir -p gpurun_out
TGB_IMPORT_TIMING=1 timeout 900 python -m pytest tests/test_gpu_import.py -m gpu -q -x -s > gpurun_out/r2im_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2im_pytest.log
