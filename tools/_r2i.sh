mkdir -p gpurun_out
# sweep launch time in four measurement modes (same generation 3 of cfg4)
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2i_launches_nocache.csv python tools/one_generation.py cfg4 16384 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_sweep_chunked --launch-skip 2 -c 1 --replay-mode application --csv --log-file gpurun_out/r2i_app_replay.csv python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_sweep_chunked --launch-skip 2 -c 1 --csv --log-file gpurun_out/r2i_kernel_replay.csv python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
timeout 600 python tools/sweep_repeat.py cfg4 16384 > gpurun_out/r2i_repeat.txt 2>&1
