mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_minkunet.py -q -x > gpurun_out/t_ac.log 2>&1; echo rc=$? >> gpurun_out/t_ac.log
tail -3 gpurun_out/t_ac.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/r02ac_layers.csv > gpurun_out/bench_ac.log 2>&1
tail -1 gpurun_out/bench_ac.log | cut -c1-200
