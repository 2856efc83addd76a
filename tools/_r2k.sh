mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ac.py -q > gpurun_out/r2k_ac.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_ac.log
