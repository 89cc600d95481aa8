mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_driver.py tests/test_gpu_validation.py tests/test_gpu_gw.py -x -q > gpurun_out/driver_tests.log 2>&1; echo "rc=$?" >> gpurun_out/driver_tests.log
TRACE_DUMP=gpurun_out/trace_si64.txt timeout 300 python tools/trace_build.py si64 30 > gpurun_out/trace_si64.log 2>&1
tail -15 gpurun_out/driver_tests.log; head -60 gpurun_out/trace_si64.log
