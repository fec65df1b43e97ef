mkdir -p gpurun_out
timeout 900 python tools/tune_minkunet.py > gpurun_out/tune_x.log 2>&1
cp paper_2204_10319_b200/configs/minkunet_b200_shapes.json gpurun_out/ 2>/dev/null
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/r02x_layers.csv > gpurun_out/bench_x.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --strategy none > gpurun_out/bench_x0.log 2>&1
tail -25 gpurun_out/tune_x.log; tail -1 gpurun_out/bench_x.log | cut -c1-300; tail -1 gpurun_out/bench_x0.log | cut -c1-300
