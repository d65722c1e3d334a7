FTN_LIBFTN=vtmp/libftn_trace.so FTN_W3_TRACE_DUMP=3 timeout 300 python tools/time3d_T.py --sweeps 24 --reps 1 --T 3 2048 > gpurun_out/w3trace2_2048.log 2>&1
FTN_LIBFTN=vtmp/libftn_trace.so FTN_W3_TRACE_DUMP=3 timeout 300 python tools/time3d_T.py --sweeps 24 --reps 1 --T 3 512 > gpurun_out/w3trace2_512.log 2>&1
for w in "12,12" "14,11" "16,11" "14,10"; do echo "== w $w"; FTN_W3_EDGE_W=$w timeout 300 python tools/time3d_T.py --sweeps 24 --reps 2 --T 3 2048 512 2>&1; done
timeout 600 python -m pytest tests/test_gpu_jacobi.py -q -x -m "gpu and not slow" -k "3d" 2>&1 | tail -1
