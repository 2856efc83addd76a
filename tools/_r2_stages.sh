mkdir -p gpurun_out
timeout 600 python bench.py --stage import --config cfg4 --steps 5 > gpurun_out/r2st_import_cfg4.json 2> gpurun_out/r2st_import_cfg4.err
timeout 600 python bench.py --stage import --config cfg2 --steps 5 > gpurun_out/r2st_import_cfg2.json 2> gpurun_out/r2st_import_cfg2.err
