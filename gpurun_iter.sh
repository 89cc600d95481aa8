mkdir -p gpurun_out
( SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 '' 'LRGW_SELECT_DEVLOOP=0'
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py c60 '' 'LRGW_SELECT_DEVLOOP=0' ) > gpurun_out/sweep_devloop.txt 2>&1
grep -v Warn gpurun_out/sweep_devloop.txt
