# correctness first, then a same-box A/B against _lib_var/$1, then the ticket trace
V=${1:-carry}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_segments.py tests/test_gpu_callers.py -m gpu -x -q 2>&1 | tail -5
bash tools/gpu_ab_enc.sh $V
bash tools/gpu_ticket_trace.sh > /dev/null 2>&1; head -40 gpurun_out/tt_alexnet.txt; sed -n 41,100p gpurun_out/tt_alexnet.txt | awk '{print $1, $2, $3, $5}' | paste -sd' ' | fold -w 200
