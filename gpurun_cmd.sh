mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py tests/test_gpu_projections.py tests/test_gpu_gw.py tests/test_gpu_dist.py -x -q -k "not si512" > gpurun_out/low_tests.log 2>&1; echo "rc=$?" >> gpurun_out/low_tests.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_low.log 2>&1
tail -3 gpurun_out/low_tests.log; grep -o '"value": [0-9.]*\|"stages_ms": {[^}]*}\|"roofline": {[^}]*}' gpurun_out/bench_low.log | head -4
