timeout 300 python tools/trace_apply2.py si64 2>&1 | grep -E "tn_|nn_|span"
timeout 600 python -m pytest tests/test_gpu_build.py tests/test_gpu_parity.py -k "apply or build" -q -x 2>&1 | tail -1
