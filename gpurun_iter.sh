mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "quadrature or node_terms or contour" 2>&1 | tail -2
# reference arm wall time at the default config
( time timeout 1500 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_default.log 2>&1 ) 2> gpurun_out/bench_reference_time.log; tail -3 gpurun_out/bench_reference_time.log; cut -c1-300 gpurun_out/bench_reference_default.log | tail -2
# launch lists: Si64 bench command, Si512 one-step bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_si64_session4.csv python bench.py --config si64 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_si64.log 2>&1; echo "ncu si64 rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_si512_session4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-implicit-line --no-pipelined-e2e > gpurun_out/ncu_launch_si512.log 2>&1; echo "ncu si512 rc=$?"
# ncu full of the TMA K3 kernel at Si512 and Si64 shapes
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad4_kernel -c 1 -f -o gpurun_out/ncu_quad4_si512 python tools/bench_quad.py si512 > gpurun_out/ncu_quad4_si512.log 2>&1; echo "ncu quad4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quad4_kernel -c 1 -f -o gpurun_out/ncu_quad4_si64 python tools/bench_quad.py si64 > gpurun_out/ncu_quad4_si64.log 2>&1; echo "ncu quad4 rc=$?"
