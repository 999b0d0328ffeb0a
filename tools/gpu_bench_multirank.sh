# Plumbing check of bench.py's N > 1 path on ONE GPU: 2 and 4 ranks over gloo
# sharing cuda:0 (NCCL refuses two ranks on one device).  Not a measurement.
for N in 2 4; do for M in allgather two_round; do
  A8_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 3 --warmup 3 --mode $M \
    > gpurun_out/mr_${N}_${M}.json 2> gpurun_out/mr_${N}_${M}.err; echo "N=$N $M rc=$?"
  head -c 400 gpurun_out/mr_${N}_${M}.json; echo; tail -3 gpurun_out/mr_${N}_${M}.err
done; done
A8_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/mr_ref.json 2>&1; echo "ref rc=$?"; head -c 300 gpurun_out/mr_ref.json
