timeout 900 python tools/tune_minkunet.py gpurun_out/shapes_new.json > gpurun_out/tune.log 2>&1; echo tune rc=$?; tail -25 gpurun_out/tune.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-110
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy gpurun_out/shapes_new.json 2>&1 | tail -1 | cut -c1-110
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy none 2>&1 | tail -1 | cut -c1-110
done
