timeout 1800 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
( SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si216 '' ) 2>&1 | grep -v Warn
TRACE_DUMP=gpurun_out/trace_si64_p4.txt timeout 300 python tools/trace_build.py si64 3 2>&1 | grep -v Warn | grep -E "panel|stages"
