mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
( SWEEP_REPS=3 timeout 900 python tools/env_sweep.py si64 ''
  SWEEP_REPS=2 timeout 900 python tools/env_sweep.py si512 '' ) > gpurun_out/sweep_smw_side.txt 2>&1
grep -v Warn gpurun_out/sweep_smw_side.txt
