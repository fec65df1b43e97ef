timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_cf.log 2>&1; echo tests; tail -2 gpurun_out/t_cf.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --layer-csv gpurun_out/r02cf_layers.csv > gpurun_out/bench_cf.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_cf.log | cut -c1-200
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_cf.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref_cf.log | cut -c1-200
timeout 600 python bench.py --model centerpoint --steps 20 --warmup 5 > gpurun_out/bench_cp_cf.log 2>&1; echo cp rc=$?; tail -1 gpurun_out/bench_cp_cf.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cf.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cf.log 2>&1; echo ncu1 rc=$?
