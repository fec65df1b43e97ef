for sh in 0 5 6 7 8; do SCB_SORT_BLOCK_SHIFT=$sh CIN=96 COUT=96 SHAPES="2:42,1:96" timeout 120 python tools/layer_probe.py 2>&1 | sed "s/^/shift=$sh /"; done
for sh in 0 6 7; do SCB_SORT_BLOCK_SHIFT=$sh CIN=64 COUT=64 LEVEL=1 SHAPES="2:42,5:48" timeout 120 python tools/layer_probe.py 2>&1 | sed "s/^/shift=$sh /"; done
