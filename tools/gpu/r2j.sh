mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jacobi.py -q -m "gpu and not slow" -x -k "3d or c5 or harmonic or random" > gpurun_out/pytest_r2j.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_r2j.log
timeout 600 python tools/time3d_T.py --sweeps 20 512 1024 2>&1
timeout 600 python tools/time3d_T.py --sweeps 100 --reps 1 2048 2>&1
FTN_J3_TB2=1 timeout 300 python tools/time3d_T.py --sweeps 100 --reps 1 --T 2 2048 2>&1
