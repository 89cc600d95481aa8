mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py tests/test_gpu_topk.py tests/test_gpu_dist.py -x -q -k "not si512" > gpurun_out/sel_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sel_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/sel_tests.log; grep -o '"value": [0-9.]*\|"stages_ms": {[^}]*}' gpurun_out/bench.log | head -3
