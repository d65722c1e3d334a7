mkdir -p gpurun_out
python tools/prof_tra.py 1024 512 512 2 > gpurun_out/plain_tra.log 2>&1 && cat gpurun_out/plain_tra.log && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:ta_ -c 8 --csv --log-file gpurun_out/ncu_tra.csv python tools/prof_tra.py 1024 512 512 2 > gpurun_out/ncu_tra.log 2>&1; echo "ncu rc=$?"
