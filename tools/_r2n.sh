mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_n.log 2>&1; echo rc=$? >> gpurun_out/t_n.log
timeout 900 python bench.py --steps 20 --warmup 5 --layer-csv gpurun_out/r02n_layers.csv > gpurun_out/bench_n.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_n.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_n.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_n.log 2>&1
tail -n 5 gpurun_out/t_n.log; tail -1 gpurun_out/bench_n.log | cut -c1-600; tail -1 gpurun_out/bench_ref_n.log | cut -c1-400
