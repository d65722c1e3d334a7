for v in base ns2 r6ns2 r2ns3 r2ns2 ns2; do
  if [ $v = base ]; then L=""; else L="vtmp/libftn_$v.so"; fi
  echo "== $v"; FTN_LIBFTN=$L timeout 300 python tools/time2d.py --reps 3 7 8 2>&1
done
