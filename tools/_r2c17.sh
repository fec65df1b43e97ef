timeout 900 python -m pytest tests/test_gpu_upscatter.py -x -q --timeout 240 > gpurun_out/t_c17.log 2>&1; echo tests; tail -15 gpurun_out/t_c17.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c17_layers.csv > gpurun_out/bench_c17.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c17.log | cut -c1-200
SCB_DENSE_K1=0 timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c17b.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c17b.log | cut -c1-200
