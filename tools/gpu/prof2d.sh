# ncu --set full of one launch of the 2-D fused kernel at several T (and the old kernel at T=5)
mkdir -p gpurun_out
for T in 5 8; do
  FTN_JACOBI_FUSE=$T ncu --set full --import-source on --clock-control none -k regex:jacobi2d_wq -s 2 -c 1 \
    -o gpurun_out/wq_T$T -f python tools/time2d.py --reps 1 $T > gpurun_out/ncu_wq_T$T.log 2>&1
done
FTN_WF_OLD=1 ncu --set full --clock-control none -k regex:jacobi2d_wf -s 2 -c 1 -o gpurun_out/wf_T5 -f \
  python tools/time2d.py --reps 1 5 > gpurun_out/ncu_wf_T5.log 2>&1
ls -la gpurun_out
