( SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py c60 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si216 ''
  SWEEP_REPS=1 timeout 900 python tools/env_sweep.py si512 '' ) 2>&1 | grep -v Warn
timeout 1500 python -m pytest tests -m gpu -x -q -rf -k "config or build or parity" > gpurun_out/gpu_tests_sub.log 2>&1; tail -2 gpurun_out/gpu_tests_sub.log
