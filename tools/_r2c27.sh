timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "epilogue or residual or minkunet" > gpurun_out/t_c27.log 2>&1; echo tests; tail -1 gpurun_out/t_c27.log
for i in 1 2 3; do SCB_LIB_NAME=libsparseconv_b200_old.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-100; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-100; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/c27_layers.csv > /dev/null 2>&1
