for q in 8 16 32 128; do echo "== qbpi $q"; SSA_VQ_QB_PER_ITEM=$q timeout 300 python tools/mq1_timing.py 4 1 2>&1 | grep -v "^  tc"; done
echo "== SSA_VQ=0"; SSA_VQ=0 timeout 300 python tools/mq1_timing.py 4 2 2>&1 | grep -v "^  tc"
