mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -x -q > gpurun_out/sketch_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sketch_tests.log
tail -25 gpurun_out/sketch_tests.log
