for ns in 0 5 10 15 20 30 40 60 80 119; do echo "nseg $ns"; FTN_WF_NSEG=$ns python tools/time_small.py 1024 1000 2>&1 | grep -E "T=(5|6) "; done
