mkdir -p gpurun_out/exp
cd $GRAFT_REPO_ROOT
SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 '' 'LRGW_SELECT_ROUND=0' 'LRGW_SELECT_ACCEPT=80' 'LRGW_SELECT_ROUND=64' > gpurun_out/exp/round_si64.log 2>&1
SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si216 '' 'LRGW_SELECT_ROUND=0' 'LRGW_SELECT_ACCEPT=80' > gpurun_out/exp/round_si216.log 2>&1
SWEEP_REPS=2 timeout 1800 python tools/env_sweep.py si512 '' 'LRGW_SELECT_ROUND=0' > gpurun_out/exp/round_si512.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -rf -x > gpurun_out/exp/parity.log 2>&1
