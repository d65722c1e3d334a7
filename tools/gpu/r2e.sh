mkdir -p gpurun_out
for W in 16 20 24 32; do echo "== edge weight $W"; FTN_WF_WQ=1 FTN_WQ_EDGE_W=$W timeout 300 python tools/time2d.py --reps 3 7 8 2>&1; done
for W in 16 24; do echo "== bigu1 w$W"; FTN_WF_WQ=1 FTN_WQ_EDGE_W=$W FTN_LIBFTN=vtmp/libftn_bigu1.so timeout 300 python tools/time2d.py --reps 3 5 7 8 9 10 2>&1; done
echo "== big w20"; FTN_WF_WQ=1 FTN_WQ_EDGE_W=20 FTN_LIBFTN=vtmp/libftn_big.so timeout 300 python tools/time2d.py --reps 3 9 10 2>&1
