mkdir -p gpurun_out
python tools/prof_adv.py 2048 1024 1024 5 > gpurun_out/plain_adv.log 2>&1 && cat gpurun_out/plain_adv.log && \
ncu --set full --import-source on --clock-control none -k regex:adv_tma -s 1 -c 1 \
    -o gpurun_out/adv -f python tools/prof_adv.py 2048 1024 1024 1 > gpurun_out/ncu_adv.log 2>&1; echo "ncu rc=$?"
