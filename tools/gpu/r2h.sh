echo "== new base (unroll 1)"; timeout 300 python tools/time2d.py --reps 3 7 8 2>&1
echo "== new u2"; FTN_LIBFTN=vtmp/libftn_u2.so timeout 300 python tools/time2d.py --reps 3 7 8 2>&1
echo "== big 9 10"; FTN_LIBFTN=vtmp/libftn_big.so timeout 300 python tools/time2d.py --reps 3 9 10 2>&1
