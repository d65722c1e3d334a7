mkdir -p gpurun_out
timeout 900 python bench.py --dist --steps 4 --warmup 3 --no-cpu > gpurun_out/bench_dist_r2x.json 2> gpurun_out/bench_dist_r2x.err; echo "bench --dist rc=$?"; tail -3 gpurun_out/bench_dist_r2x.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r2x.json 2> gpurun_out/bench_ref_r2x.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_r2x.json | head -c 1200; echo
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
