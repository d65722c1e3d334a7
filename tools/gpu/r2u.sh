for v in base st256 base st256; do
  if [ $v = base ]; then L=""; else L="vtmp/libftn_$v.so"; fi
  echo "== $v"; FTN_LIBFTN=$L timeout 300 python tools/time2d.py --reps 3 8 2>&1
done
