mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_s.log 2>&1; echo rc=$? >> gpurun_out/t_s.log
CIN=96 COUT=96 timeout 300 python tools/layer_probe.py > gpurun_out/probe_s.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/r02s_layers.csv > gpurun_out/bench_s.log 2>&1
tail -n 5 gpurun_out/t_s.log; cat gpurun_out/probe_s.log; tail -1 gpurun_out/bench_s.log | cut -c1-400
