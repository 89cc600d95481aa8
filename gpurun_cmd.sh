python -c "
import cProfile, pstats, sys, os
sys.argv=['dist_time.py','--config','si64','--reps','2']
sys.path.insert(0,'tools')
import dist_time
cProfile.run('dist_time.main()','gpurun_out/dist.prof')
p=pstats.Stats('gpurun_out/dist.prof'); p.sort_stats('tottime').print_stats(25)
" 2>&1 | tail -45
