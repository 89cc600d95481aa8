mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py -x -q > gpurun_out/had_tests.log 2>&1; echo "rc=$?" >> gpurun_out/had_tests.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_had.log 2>&1
LRGW_HAD_TALL=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_had0.log 2>&1
timeout 600 python tools/trace_build.py si512 3 > gpurun_out/trace_si512_had.log 2>&1
tail -3 gpurun_out/had_tests.log; for f in bench_had bench_had0; do grep -o '"value": [0-9.]*\|"stages_ms": {[^}]*}' gpurun_out/$f.log | head -3; done; grep -E "stages|hadamard|Gemm2Cfg<64, (48|64|80|96|112|128), 16, (48|64|80|96|112|128), 3, 2, true" gpurun_out/trace_si512_had.log | head -12
