C=paper_2204_10319_b200/configs
for i in 1 2; do
for cfg in "1 _new" "1 _old" "0 _old" "0 _new" "1 none" "0 none"; do set -- $cfg
  S=$C/${2}_shapes.json; [ "$2" = none ] && S=none
  SCB_IC_RING=$1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --strategy $S > gpurun_out/bench_ax_$1$2$i.log 2>&1
done; done
for f in gpurun_out/bench_ax_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$f\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; done
