timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_aq.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t_aq.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --layer-csv gpurun_out/r02aq_layers.csv > gpurun_out/bench_aq.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_aq.log 2>&1; echo ref rc=$?
timeout 600 python bench.py --model centerpoint --steps 20 --warmup 5 > gpurun_out/bench_cp_aq.log 2>&1; echo cp rc=$?
