for v in base blkold; do
  if [ $v = base ]; then lib=paper_1511_04561_b200/_lib/libapprox8_b200.so; else lib=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so; fi
  echo "== $v"; A8_LIB=$lib timeout 300 python tools/sweep_blocked.py 2>&1 | tail -4; A8_LIB=$lib timeout 300 python tools/prof_blocked.py 2>&1 | tail -2
done
