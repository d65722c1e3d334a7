mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tra_adv.py -q -x > gpurun_out/pytest_tra4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_tra4.log
python tools/prof_tra.py 1024 512 512 20
FTN_TA_TMA=0 python tools/prof_tra.py 1024 512 512 20
python tools/prof_tra.py 1024 512 512 2 > gpurun_out/plain_tra.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ta_ -c 2 --csv --log-file gpurun_out/ncu_tra3.csv python tools/prof_tra.py 1024 512 512 2 > gpurun_out/ncu_tra.log 2>&1; echo "ncu rc=$?"
