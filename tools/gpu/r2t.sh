for b in 1 0 8 32; do
  if [ $b = 0 ]; then E=""; else E="FTN_WQ_BANDS=$b"; fi
  echo "== bands $b"; env $E timeout 300 python tools/time2d.py --reps 3 8 2>&1
done
timeout 600 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_solve.py -q -x -m "gpu and not slow" 2>&1 | tail -1
