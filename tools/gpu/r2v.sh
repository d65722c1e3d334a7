FTN_LIBFTN=vtmp/libftn_trace.so FTN_W3_TRACE_DUMP=3 timeout 300 python tools/time3d_T.py --sweeps 24 --reps 1 --T 3 2048 > gpurun_out/w3trace_2048.log 2>&1
FTN_LIBFTN=vtmp/libftn_trace.so FTN_W3_TRACE_DUMP=3 timeout 300 python tools/time3d_T.py --sweeps 24 --reps 1 --T 3 512 > gpurun_out/w3trace_512.log 2>&1
ls -la gpurun_out/w3trace*
