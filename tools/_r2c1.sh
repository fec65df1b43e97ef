timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_c1.log 2>&1; echo tests; tail -3 gpurun_out/t_c1.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_c1.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_c1.log
