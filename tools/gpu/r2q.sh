for v in base nw16 nw16ns6; do
  if [ $v = base ]; then L=""; else L="vtmp/libftn_$v.so"; fi
  echo "== $v"; FTN_LIBFTN=$L timeout 300 python tools/time3d_T.py --sweeps 24 --reps 2 --T 3,4 2048 2>&1
done
FTN_LIBFTN=vtmp/libftn_nw16.so timeout 300 python -m pytest tests/test_gpu_jacobi.py -q -x -k "3d" 2>&1 | tail -1
