mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_jacobi.py -q -m "gpu and not slow" -x -k "3d or c5 or harmonic or random" > gpurun_out/pytest_r2l.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2l.log
timeout 600 python tools/time3d_T.py --sweeps 20 1024 2>&1
timeout 600 python tools/time3d_T.py --sweeps 100 --reps 1 2048 2>&1
python tools/time3d_T.py --sweeps 8 --reps 1 --T 4 1024 > gpurun_out/plain_wr4b.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:jacobi3d_wr -s 1 -c 1 \
    -o gpurun_out/wr4b -f python tools/time3d_T.py --sweeps 8 --reps 1 --T 4 1024 > gpurun_out/ncu_wr4b.log 2>&1; echo "ncu rc=$?"
