export A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so
echo "=== sched0"; timeout 300 python tools/ticket_timeline.py 2>&1 | tail -9
echo "=== sched1"; A8_SCHED=1 timeout 300 python tools/ticket_timeline.py 2>&1 | tail -9
