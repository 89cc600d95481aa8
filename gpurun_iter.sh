mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
( SWEEP_REPS=2 timeout 900 python tools/env_sweep.py c60 '' 'LRGW_PANEL=0' 'LRGW_PANEL=1'
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si216 '' 'LRGW_PANEL=0' 'LRGW_PANEL=1' ) > gpurun_out/sweep_panel_c60_si216.txt 2>&1
tail -3 gpurun_out/gpu_tests.log; grep -v Warn gpurun_out/sweep_panel_c60_si216.txt
