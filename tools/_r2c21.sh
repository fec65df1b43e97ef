for a in 2 4; do for d in 0 15; do SCB_UP_NACC=$a SCB_UP_DEBUG=$d EPI=1 L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo "nacc=$a debug=$d"; done; done
