mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_build.py -x -q -k "not si512" > gpurun_out/pd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pd_tests.log
tail -n 3 gpurun_out/pd_tests.log
