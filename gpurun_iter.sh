( SWEEP_REPS=2 timeout 1200 python tools/env_sweep.py si512 '' 'LRGW_SELECT_ACCEPT=96'
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si64 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si216 '' 'LRGW_SELECT_ACCEPT=96' ) 2>&1 | grep -v Warn
