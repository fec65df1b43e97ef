timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "epilogue or residual or pair or fused" > gpurun_out/t_c16.log 2>&1; echo tests; tail -2 gpurun_out/t_c16.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c16_layers.csv > gpurun_out/bench_c16.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c16.log | cut -c1-200
