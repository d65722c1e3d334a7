nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_throttle_reasons.active --format=csv,noheader -lms 200 > gpurun_out/r2ao_smi.csv &
SMI=$!
sleep 1; echo "idle mark"; date +%s.%N
timeout 300 python tools/time3d_T.py --sweeps 48 --reps 3 --T 3 2048 2>&1 | tail -1; date +%s.%N
FTN_LIBFTN=vtmp/libftn_w12L.so timeout 300 python tools/time3d_T.py --sweeps 48 --reps 3 --T 3 2048 2>&1 | tail -1; date +%s.%N
timeout 300 python tools/time2d.py 2>&1 | tail -2; date +%s.%N
kill $SMI
