timeout 600 python -m pytest tests/test_gpu_reorder.py tests/test_gpu_minkunet.py tests/test_gpu_fullsize.py tests/test_gpu_centerpoint.py -q -x 2>&1 | tail -1
for cfg in "96 96 0" "32 32 0" "64 64 1"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 SHAPES="2:0,1:0" timeout 120 python tools/layer_probe.py 2>&1 | sed "s/^/$1->$2 L$3 /" | cut -c1-150; done
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bd$i.log 2>&1; done
for f in gpurun_out/bench_bd?.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$f\", round(d[\"value\"],1), round(d[\"e2e\"][\"value\"],1))"; done
