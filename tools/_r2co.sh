timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "pair or fused or minkunet or epilogue" > gpurun_out/t_co.log 2>&1; echo tests; tail -1 gpurun_out/t_co.log
for i in 1 2 3; do SCB_IC_SMALL_LEVEL=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-100; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-100; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/co_layers.csv > /dev/null 2>&1
SCB_IC_SMALL_LEVEL=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/co0_layers.csv > /dev/null 2>&1
