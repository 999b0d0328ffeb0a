for wf in 2000 6432; do
echo "== A8_SCHED_FILL=$wf"
A8_SCHED_FILL=$wf A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so timeout 300 python tools/switch_trace.py 2>&1 | tail -25
done
