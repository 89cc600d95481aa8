timeout 900 python -m pytest tests/test_gpu_topk.py -x -q -rf 2>&1 | tail -3
( SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si512 '' ) 2>&1 | grep -v Warn
