timeout 900 python -m pytest tests/test_gpu_trtri.py tests/test_gpu_build.py tests/test_gpu_implicit.py -x -q 2>&1 | tail -2
( SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py c60 '' ) 2>&1 | grep -v Warn | cut -c1-160
