mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log
python tools/prof_build.py > gpurun_out/plain_prof.log 2>&1 && \
ncu --nvtx --print-nvtx-rename kernel --profile-from-start off --csv --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --log-file gpurun_out/traffic.csv python tools/prof_build.py > gpurun_out/ncu_traffic.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:dgemm3_kernel -c 1 \
    -o gpurun_out/prof_pvp python tools/prof_build.py > gpurun_out/ncu_pvp.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/bench_final.log | cut -c1-400; tail -3 gpurun_out/ncu_pvp.log
