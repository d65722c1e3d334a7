for n in 8192 4096 2048 1024; do
  sw=100; [ $n -le 2048 ] && sw=1000
  echo "== n=$n wf/wq default"; FTN_WQ_EDGE_W=16 timeout 300 python tools/time2d.py --n $n --sweeps $sw --reps 3 5 6 7 8 2>&1
  echo "== n=$n all wq"; FTN_WF_WQ=1 FTN_WQ_EDGE_W=16 timeout 300 python tools/time2d.py --n $n --sweeps $sw --reps 3 4 5 6 2>&1
done
