timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reorder.py -q -x 2>&1 | tail -1
for cfg in "96 96 0" "32 32 0" "8 32 0" "64 64 1" "128 128 2" "256 256 3" "96 96 1"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 SHAPES="2:0,3:24,2:42,1:0" timeout 120 python tools/layer_probe.py 2>&1 | sed "s/^/$1->$2 L$3 /" | cut -c1-120; done
