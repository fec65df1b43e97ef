timeout 900 python -m pytest tests/test_gpu_upscatter.py -x -q --timeout 240 > gpurun_out/t_c18.log 2>&1; echo tests; tail -15 gpurun_out/t_c18.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c18_layers.csv > gpurun_out/bench_c18.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c18.log | cut -c1-200
