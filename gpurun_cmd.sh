mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/dist_time.py --config si64 > gpurun_out/dist_time_si64.log 2>&1
timeout 300 python -c "
import cProfile, pstats, sys, os
sys.argv=['dist_time.py','--config','si64','--reps','2']
sys.path.insert(0,'tools')
import dist_time
cProfile.run('dist_time.main()', 'gpurun_out/dist.prof')
p=pstats.Stats('gpurun_out/dist.prof'); p.sort_stats('tottime').print_stats(35)
" > gpurun_out/dist_profile.log 2>&1
tail -4 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -20 gpurun_out/dist_time_si64.log
