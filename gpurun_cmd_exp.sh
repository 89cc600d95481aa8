mkdir -p gpurun_out/prof
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/prof/bench_si512.log 2>&1
timeout 300 python tools/prof_build.py si64 > gpurun_out/prof/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_si64.csv python tools/prof_build.py si64 > gpurun_out/prof/ncu_launch.log 2>&1
ncu --nvtx --print-nvtx-rename kernel --profile-from-start off --csv --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --log-file gpurun_out/prof/traffic_si64.csv python tools/prof_build.py si64 > gpurun_out/prof/ncu_traffic.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:dgemm4k -c 1 -o gpurun_out/prof/pvp_si64 python tools/prof_build.py si64 > gpurun_out/prof/ncu_pvp.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:dgemm4_kernel -c 1 -o gpurun_out/prof/fit_si64 python tools/prof_build.py si64 > gpurun_out/prof/ncu_fit.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"cand_greedy|dgemm2_kernel" -c 4 -o gpurun_out/prof/select_si64 python tools/prof_build.py si64 > gpurun_out/prof/ncu_select.log 2>&1
timeout 900 python tools/prof_build.py si512 > gpurun_out/prof/plain512.log 2>&1 && \
ncu --nvtx --print-nvtx-rename kernel --profile-from-start off --csv --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"dgemm4k|dgemm4_kernel|quad_kernel" --log-file gpurun_out/prof/traffic_si512.csv python tools/prof_build.py si512 > gpurun_out/prof/ncu_traffic512.log 2>&1
ls -la gpurun_out/prof
