export A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so
echo "=== premax"; A8_PREMAX=1 timeout 300 python tools/ticket_timeline.py 2>&1 | tail -8
unset A8_LIB
for h in 0 2 4 8 16; do echo "hold $h"; A8_PREMAX_HOLD=$h timeout 300 python tools/prof_codec.py --case alexnet --premax 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_premax.py -q 2>&1 | tail -2
