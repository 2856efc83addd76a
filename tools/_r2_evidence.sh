# Round-2 evidence: bench lines for every config (DC + AC stage), the reference
# arm, launch lists and ncu --set full of the top kernels.  usage: bash tools/_r2_evidence.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
for c in cfg4 cfg2 cfg1 cfg3; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
for c in cfg1 ac118; do
  timeout 600 python bench.py --stage ac --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_ac_$c.json 2> gpurun_out/${TAG}_bench_ac_$c.err
done
for c in cfg4 cfg2 cfg1; do
  B=$(python -c "from bench import CONFIGS; print(CONFIGS['$c']['batch'])")
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_${TAG}.csv python tools/one_generation.py $c $B 5 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_${c}_${TAG}.csv > gpurun_out/launches_${c}_${TAG}_summary.txt
done
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o gpurun_out/chunked_cfg4_${TAG} python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
$NCU -k regex:"k_prep_rows|k_finish" --launch-skip 8 -c 4 -o gpurun_out/prepfin_cfg4_${TAG} python tools/step_timing.py cfg4 16384 > /dev/null 2>&1
$NCU -k regex:k_sweep_chunked --launch-skip 4 -c 1 -o gpurun_out/chunked_cfg2_${TAG} python tools/step_timing.py cfg2 4096 > /dev/null 2>&1
timeout 600 python bench.py --stage import --config cfg4 --steps 5 > gpurun_out/${TAG}_bench_import_cfg4.json 2> gpurun_out/${TAG}_bench_import_cfg4.err
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
