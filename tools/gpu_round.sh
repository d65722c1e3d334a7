#!/bin/bash
# One GPU call: parity tests, the bench line, the launch list and an ncu --set full capture
# of the top kernels.  Usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --rows none --no-cpu > gpurun_out/bench_small_$tag.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 2 --warmup 1 --rows none --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
python tools/prof_case.py all > gpurun_out/prof_plain_$tag.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"jacobi2d_wq|jacobi2d_wf|jacobi2d_tma|jacobi3d_wr|jacobi3d_tma|jacobi3d_tb2|reduce_chunks|transpose_kernel|dmma_gemm|ew_kernel<double, 5|vec|adv_tma" -c 30 \
  -o gpurun_out/prof_$tag python tools/prof_case.py all > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu full rc=$?"
# summarise on the box (gpurun copies back at most 64 MiB): the summary always, the report only if small
python tools/ncu_summary.py full gpurun_out/prof_$tag.ncu-rep > gpurun_out/full_top_$tag.txt 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_$tag.csv > gpurun_out/launches_summary_$tag.txt 2>&1
[ $(stat -c %s gpurun_out/prof_$tag.ncu-rep 2>/dev/null || echo 0) -gt 40000000 ] && mv gpurun_out/prof_$tag.ncu-rep /tmp/
du -sh gpurun_out
