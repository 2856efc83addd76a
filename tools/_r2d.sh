mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prep --launch-skip 3 -c 1 -o gpurun_out/prep_cfg4_r2v2 python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o gpurun_out/chunked_cfg4_r2v2 python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
