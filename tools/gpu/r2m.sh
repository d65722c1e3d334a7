for w in 8 12 16 24; do echo "== edge w $w"; FTN_W3_EDGE_W=$w timeout 300 python tools/time3d_T.py --sweeps 24 --reps 2 --T 3,4 2048 2>&1; done
