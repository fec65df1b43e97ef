run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cl_$tag.log 2>&1; tail -1 gpurun_out/cl_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$tag\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; }
for i in 1 2 3; do
run base$i X=1
run prio0_$i SCB_MAP_PRIORITY=0
run lvl3_$i SCB_PREFETCH_LEVEL=3
run p0l3_$i SCB_MAP_PRIORITY=0 SCB_PREFETCH_LEVEL=3
done
