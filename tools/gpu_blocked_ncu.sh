mkdir -p gpurun_out
for b in 4096 1024; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"blocked_encode_stream" -s 2 -c 1 -o gpurun_out/full_blocked_$b python tools/prof_blocked_one.py 28 $b > /dev/null 2>&1; echo ncu=$?
done
