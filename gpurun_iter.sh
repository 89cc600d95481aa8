( SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 '' 'LRGW_TMA_PERSIST=0'
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py c60 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si216 ''
  SWEEP_REPS=2 timeout 1200 python tools/env_sweep.py si512 '' ) 2>&1 | grep -v Warn | cut -c1-110
