mkdir -p gpurun_out
FTN_WF_WQ=1 timeout 600 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_solve.py tests/test_gpu_virtual_ranks.py -x -q -m "gpu and not slow" > gpurun_out/pytest_r2d.log 2>&1; echo "pytest wq rc=$?"; tail -3 gpurun_out/pytest_r2d.log
for W in 8 12 16; do echo "== edge weight $W"; FTN_WF_WQ=1 FTN_WQ_EDGE_W=$W timeout 300 python tools/time2d.py --reps 3 5 6 7 8 2>&1; done
for v in m2 m2ns4; do echo "== $v"; FTN_WF_WQ=1 FTN_LIBFTN=vtmp/libftn_$v.so timeout 300 python tools/time2d.py --reps 3 4 5 6 2>&1; done
echo "== wf default"; timeout 120 python tools/time2d.py --reps 3 5 2>&1
