# cfg1 / QD check: replay tests, cfg1 bench, launch list; $1 = tag
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qd.py -m gpu -q -x > gpurun_out/$1_qd_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$1_qd_pytest.log
timeout 400 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/$1_bench_cfg1.json 2> gpurun_out/$1_bench_cfg1.err
B=$(python -c "from bench import CONFIGS; print(CONFIGS['cfg1']['batch'])")
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1_$1.csv python tools/one_generation.py cfg1 $B 5 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg1_$1.csv > gpurun_out/launches_cfg1_$1_summary.txt
