# Plumbing check of bench.py's N > 1 path on ONE GPU: ranks over gloo sharing
# cuda:0 (NCCL refuses two ranks on one device).  Not a measurement.
mkdir -p gpurun_out
for cfg in "2 allgather" "2 two_round" "4 two_round"; do set -- $cfg; N=$1; M=$2
  A8_BENCH_BACKEND=gloo timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 3 --warmup 3 --mode $M \
    > gpurun_out/mr_${N}_${M}.json 2> gpurun_out/mr_${N}_${M}.err; echo "N=$N $M rc=$?"
  head -c 1500 gpurun_out/mr_${N}_${M}.json; echo; grep -v "^W1\|^\*\|OMP" gpurun_out/mr_${N}_${M}.err | tail -5
done
A8_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/mr_ref.json 2>&1; echo "ref rc=$?"; head -c 300 gpurun_out/mr_ref.json
