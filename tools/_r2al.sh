mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_al.log 2>&1; echo rc=$? >> gpurun_out/t_al.log
tail -3 gpurun_out/t_al.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_al.log 2>&1
tail -1 gpurun_out/bench_al.log | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
