for v in "0 0" "8 0" "0 64" "8 64"; do set -- $v; SCB_IC_DEBUG=$1 SCB_IC_KC=$2 CIN=96 COUT=96 SHAPES="2:0,2:42,2:56,1:96,3:24" timeout 120 python tools/layer_probe.py 2>&1 | sed "s/^/dbg=$1 kc=$2 /"; done
for v in "0 0" "8 0"; do set -- $v; SCB_IC_DEBUG=$1 CIN=32 COUT=32 SHAPES="2:0,3:24" timeout 120 python tools/layer_probe.py 2>&1 | sed "s/^/dbg=$1 /"; done
