for v in base smx base smx; do
  if [ $v = base ]; then L=""; else L="vtmp/libftn_$v.so"; fi
  echo "== $v"; FTN_LIBFTN=$L timeout 300 python tools/time2d.py --reps 3 8 2>&1
done
FTN_LIBFTN=vtmp/libftn_smx.so timeout 300 python -m pytest tests/test_gpu_jacobi.py -q -x -k "2d_temporal" 2>&1 | tail -1
