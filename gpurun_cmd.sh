mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wfn1.py tests/test_dropin.py tests/test_gpu_gw.py -x -q > gpurun_out/wfn1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wfn1_tests.log
tail -30 gpurun_out/wfn1_tests.log
