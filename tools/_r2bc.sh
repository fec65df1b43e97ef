timeout 900 python tools/tune_minkunet.py gpurun_out/minkunet_b200_shapes_bc.json > gpurun_out/tune_bc.log 2>&1; tail -1 gpurun_out/tune_bc.log
cp gpurun_out/minkunet_b200_shapes_bc.json paper_2204_10319_b200/configs/_bc.json
for i in 1 2; do
SCB_IC_NP8=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy paper_2204_10319_b200/configs/_bc.json > gpurun_out/bench_bc_new$i.log 2>&1
SCB_IC_NP8=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bc_cur$i.log 2>&1
SCB_IC_NP8=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bc_np0$i.log 2>&1
done
for f in gpurun_out/bench_bc_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$f\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; done
