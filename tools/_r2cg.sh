timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_cg.log 2>&1; echo tests; tail -2 gpurun_out/t_cg.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --layer-csv gpurun_out/r02cg_layers.csv > gpurun_out/bench_cg.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_cg.log | cut -c1-200
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_cg.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref_cg.log | cut -c1-200
timeout 600 python bench.py --model centerpoint --steps 20 --warmup 5 > gpurun_out/bench_cp_cg.log 2>&1; echo cp rc=$?; tail -1 gpurun_out/bench_cp_cg.log | cut -c1-200
