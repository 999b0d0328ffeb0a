# A/B of the two encoders on one GPU: ticket (persistent) vs split (two-pass).
mkdir -p gpurun_out
out=gpurun_out/ab_encode.jsonl; : > $out
for mode in ticket split; do
  for spec in dynamic-tree/absmax mantissa/decade+1; do
    A8_ENC=$mode timeout 300 python tools/prof_codec.py --case alexnet --spec $spec | sed "s/^/{\"mode\":\"$mode\",\"keep\":0,\"r\":/; s/$/}/" >> $out
    A8_ENC=$mode timeout 300 python tools/prof_codec.py --case big --spec $spec | sed "s/^/{\"mode\":\"$mode\",\"keep\":0,\"r\":/; s/$/}/" >> $out
  done
done
for keep in 40 70 100; do
  A8_ENC=split A8_L2_KEEP_MB=$keep timeout 300 python tools/prof_codec.py --case alexnet | sed "s/^/{\"mode\":\"split\",\"keep\":$keep,\"r\":/; s/$/}/" >> $out
done
cat $out
