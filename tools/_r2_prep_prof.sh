# ncu --set full of k_prep_rows<5, 7> at cfg4: $1 = tag
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_prep_rows<.int.5" --launch-skip 5 -c 1 \
  -o gpurun_out/prep57_cfg4_$1 python tools/step_timing.py cfg4 16384 > gpurun_out/prep57_$1.log 2>&1
