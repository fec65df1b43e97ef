timeout 600 python -m pytest tests/test_gpu_upscatter.py tests/test_gpu_reorder.py -x -q > gpurun_out/t_c2.log 2>&1; echo tests; tail -15 gpurun_out/t_c2.log
for u in 0 1; do for r in 0 1; do SCB_UPSCATTER=$u L1_REORDER=$r timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo "upscatter=$u"; done; done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c2_layers.csv > gpurun_out/bench_c2.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c2.log | cut -c1-400
SCB_UPSCATTER=0 timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_off.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c2_off.log | cut -c1-300
