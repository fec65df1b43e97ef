for i in 1 2 3; do
SCB_LIB_NAME=libsparseconv_b200_old.so EPI=1 L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo old
EPI=1 L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo new
done
