timeout 900 python -m pytest tests/test_gpu_upscatter.py tests/test_gpu_reorder.py -x -q --timeout 240 -v > gpurun_out/t_c3.log 2>&1; echo tests; grep -E "PASS|FAIL|Timeout|Error|passed|failed" gpurun_out/t_c3.log | tail -25
for u in 0 1; do SCB_UPSCATTER=$u L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo "upscatter=$u"; done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c3_layers.csv > gpurun_out/bench_c3.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c3.log | cut -c1-300
