for v in base u1 u4 r2 m4 r8; do
  if [ $v = base ]; then L=""; else L="vtmp/libftn_$v.so"; fi
  echo "== $v"; FTN_LIBFTN=$L python tools/time2d.py --reps 3 3 4 5 6 7 8 2>&1
done
FTN_JACOBI_FUSE=5 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_wq -s 2 -c 1 \
    -o gpurun_out/wq2_T5 -f python tools/time2d.py --reps 1 5 > gpurun_out/ncu_wq2_T5.log 2>&1
