timeout 900 python -m pytest tests/test_gpu_upscatter.py -x -q --timeout 240 > gpurun_out/t_c10.log 2>&1; echo tests; tail -2 gpurun_out/t_c10.log
for u in 0 1; do for e in 0 1; do EPI=$e SCB_UPSCATTER=$u L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; done; done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c10_layers.csv > gpurun_out/bench_c10.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c10.log | cut -c1-200
