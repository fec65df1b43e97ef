for d in 0 16 15 31; do SCB_UP_DEBUG=$d EPI=1 SCB_UPSCATTER=1 L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo "debug=$d"; done
