mkdir -p gpurun_out
SWEEP_REPS=4 timeout 900 python tools/env_sweep.py si64 '' 'LRGW_TMA_MNSTAGES=6' 'LRGW_TMA_KSTAGES=6' 'LRGW_TMA_KSTAGES=7' 2>&1 | cut -c1-200 | tee gpurun_out/sweep_stages_si64.log
SWEEP_REPS=2 timeout 1500 python tools/env_sweep.py si512 '' 'LRGW_TMA_MNSTAGES=6 LRGW_TMA_KSTAGES=7' 'LRGW_TMA_KSTAGES=6' 2>&1 | cut -c1-200 | tee gpurun_out/sweep_stages_si512.log
