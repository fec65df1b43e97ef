timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reorder.py -q -x 2>&1 | tail -1
for np in 1 0; do for cfg in "64 64 1" "128 128 2" "256 256 3" "96 96 0" "128 256 4"; do set -- $cfg; SCB_IC_NP8=$np CIN=$1 COUT=$2 LEVEL=$3 SHAPES="1:0,2:0" timeout 120 python tools/layer_probe.py 2>&1 | grep shape | sed "s/^/np8=$np $1->$2 L$3 /"; done; done
