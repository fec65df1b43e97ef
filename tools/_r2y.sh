mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_minkunet.py tests/test_gpu_reorder.py tests/test_gpu_pair.py tests/test_gpu_reference_models.py -q -x > gpurun_out/t_y.log 2>&1; echo rc=$? >> gpurun_out/t_y.log
tail -3 gpurun_out/t_y.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/r02y_layers.csv > gpurun_out/bench_y.log 2>&1
SCB_MAP_STREAM=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_y0.log 2>&1
tail -1 gpurun_out/bench_y.log | cut -c1-250; tail -1 gpurun_out/bench_y0.log | cut -c1-250
