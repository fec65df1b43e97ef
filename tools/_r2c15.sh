timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_c15.log 2>&1; echo tests; tail -3 gpurun_out/t_c15.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --layer-csv gpurun_out/r02c_layers.csv > gpurun_out/bench_c15.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c15.log | cut -c1-250
timeout 600 python bench.py --model centerpoint --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cp_c15.log 2>&1; echo cp rc=$?; tail -1 gpurun_out/bench_cp_c15.log | cut -c1-250
