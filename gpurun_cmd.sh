mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py tests/test_gpu_topk.py tests/test_gpu_projections.py -x -q > gpurun_out/g3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g3_tests.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g3.log 2>&1
tail -n 2 gpurun_out/g3_tests.log; grep -o '"value": [0-9.]*\|"select": [0-9.]*' gpurun_out/bench_g3.log | head -3
