for i in 1 2; do for r in 0 2 1; do SCB_IC_CTAS_RULE=$r timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ba_$r$i.log 2>&1; done; done
for f in gpurun_out/bench_ba_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$f\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; done
