ITERS=40 timeout 300 python tools/pair_stress2.py 2>&1 | tail -1
SHAPES=1:0,2:0,3:24,2:42 ITERS=40 timeout 300 python tools/pair_stress2.py 2>&1 | tail -1
timeout 900 python tools/tune_minkunet.py gpurun_out/minkunet_b200_shapes_au.json > gpurun_out/tune_au.log 2>&1; tail -2 gpurun_out/tune_au.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy gpurun_out/minkunet_b200_shapes_au.json > gpurun_out/bench_au_new$i.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy none > gpurun_out/bench_au_none$i.log 2>&1
done
for f in gpurun_out/bench_au_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$f\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; done
