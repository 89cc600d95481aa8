mkdir -p gpurun_out/exp
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/exp/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/exp/gpu_all.log
SWEEP_REPS=3 timeout 600 python tools/env_sweep.py si64 '' > gpurun_out/exp/smw_si64.log 2>&1
