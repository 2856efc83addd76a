# ncu --set full of the chunked sweep and the rank 5-7 prep at cfg4: $1 = tag
mkdir -p gpurun_out
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o gpurun_out/chunked_cfg4_$1 python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
$NCU -k regex:k_prep_rows --launch-skip 7 -c 1 -o gpurun_out/prep_cfg4_$1 python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
