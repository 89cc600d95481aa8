# Round-2 verification on one B200: GPU tests, smoke, bench lines (Si512 default, Si64, C60, Si216),
# the Si64 launch list and an ncu capture of the selection panel kernel.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_si512.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si512.log
timeout 600 python bench.py --config si64 --steps 20 --warmup 5 > gpurun_out/bench_si64.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si64.log
timeout 600 python bench.py --config c60 --steps 5 --warmup 3 > gpurun_out/bench_c60.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c60.log
timeout 900 python bench.py --config si216 --steps 5 --warmup 3 > gpurun_out/bench_si216.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si216.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_si64.csv python bench.py --config si64 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel4_kernel -s 6 -c 1 -o gpurun_out/ncu_panel4_si64 python tools/trace_build.py si64 2 > gpurun_out/ncu_panel4.log 2>&1
tail -n 3 gpurun_out/gpu_tests.log; tail -n 2 gpurun_out/smoke.log; grep -h '"value"' gpurun_out/bench_*.log | cut -c1-150
