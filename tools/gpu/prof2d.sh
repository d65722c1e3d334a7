# ncu --set full of one launch of the 2-D fused kernels: wf<5> (default), wq<5>, wq<8>
mkdir -p gpurun_out
python tools/time2d.py --reps 1 5 > gpurun_out/plain_wf5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:jacobi2d_wf -s 2 -c 1 \
    -o gpurun_out/wf_T5 -f python tools/time2d.py --reps 1 5 > gpurun_out/ncu_wf_T5.log 2>&1
FTN_WF_WQ=1 python tools/time2d.py --reps 1 5 > gpurun_out/plain_wq5.log 2>&1 && \
FTN_WF_WQ=1 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_wq -s 2 -c 1 \
    -o gpurun_out/wq_T5 -f python tools/time2d.py --reps 1 5 > gpurun_out/ncu_wq_T5.log 2>&1
python tools/time2d.py --reps 1 8 > gpurun_out/plain_wq8.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:jacobi2d_wq -s 2 -c 1 \
    -o gpurun_out/wq_T8 -f python tools/time2d.py --reps 1 8 > gpurun_out/ncu_wq_T8.log 2>&1
ls -la gpurun_out
