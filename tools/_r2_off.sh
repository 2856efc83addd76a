mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_offspring --launch-skip 5 -c 1 -o gpurun_out/offspring_cfg1_r2 python tools/one_generation.py cfg1 64 7 > /dev/null 2>&1
