timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "serving or minkunet or prefetch" > gpurun_out/t_cm.log 2>&1; echo tests; tail -1 gpurun_out/t_cm.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-100; done
