mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_dist.py tests/test_gpu_parity.py -x -q -k "not si512" > gpurun_out/sk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sk_tests.log
timeout 300 python tools/dist_time.py --config si64 > gpurun_out/dist_time_si64.log 2>&1
tail -n 2 gpurun_out/sk_tests.log; tail -n 1 gpurun_out/dist_time_si64.log | cut -c1-200
