mkdir -p gpurun_out
python tools/time3d_T.py --sweeps 4 --reps 1 --T 4 1024 > gpurun_out/plain_wr4.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:jacobi3d_wr -s 1 -c 1 \
    -o gpurun_out/wr4 -f python tools/time3d_T.py --sweeps 4 --reps 1 --T 4 1024 > gpurun_out/ncu_wr4.log 2>&1; echo "ncu rc=$?"
