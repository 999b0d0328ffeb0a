export A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so
echo "=== premax"; A8_PREMAX=1 timeout 300 python tools/ticket_timeline.py 2>&1 | tail -12
