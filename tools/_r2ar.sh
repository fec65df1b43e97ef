timeout 300 python -m pytest tests/test_gpu_pair.py -q 2>&1 | tail -1
cp paper_2204_10319_b200/configs/minkunet_b200_shapes.json /tmp/old_shapes.json
timeout 900 python tools/tune_minkunet.py gpurun_out/minkunet_b200_shapes_ar.json > gpurun_out/tune_ar.log 2>&1; tail -3 gpurun_out/tune_ar.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy /tmp/old_shapes.json > gpurun_out/bench_ar_old$i.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy gpurun_out/minkunet_b200_shapes_ar.json > gpurun_out/bench_ar_new$i.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy none > gpurun_out/bench_ar_none$i.log 2>&1
done
for f in gpurun_out/bench_ar_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$f\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; done
