for v in u4 u2 u6; do
  export A8_LIB=paper_1511_04561_b200/_lib_var/$v/libapprox8_b200.so
  echo "variant=$v"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:onebit_stats -s 3 -c 2 --csv python tools/prof_onebit_c3.py 2>/dev/null | grep gpu__time | awk -F'","' '{print $NF}'
  python tools/prof_onebit_c3.py
done
