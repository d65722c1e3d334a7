for a in 1 0 1 0; do echo "== align $a"; FTN_WQ_ALIGN=$a timeout 300 python tools/time2d.py --reps 3 8 2>&1; done
timeout 300 python -m pytest tests/test_gpu_jacobi.py -q -x -k "2d_temporal" 2>&1 | tail -1
python tools/time2d.py --reps 1 8 > gpurun_out/plain_al.log 2>&1 && ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:jacobi2d_wq -s 2 -c 1 --csv python tools/time2d.py --reps 1 8 2>/dev/null | tail -4
