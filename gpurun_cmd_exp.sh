mkdir -p gpurun_out/tma3
cd $GRAFT_REPO_ROOT
for s in smw contour isdf elliptic linalg model; do (cd /tmp && timeout 600 $GRAFT_REPO_ROOT/tests/cpp/_ref/ref_test_$s > $GRAFT_REPO_ROOT/gpurun_out/tma3/ref_test_$s.log 2>&1; echo rc=$? >> $GRAFT_REPO_ROOT/gpurun_out/tma3/ref_test_$s.log); done
for k in 0 1 2; do for s in "1024 230400" "3456 746496" "8192 200000"; do LRGW_TMA_KCFG=$k timeout 120 python tools/bench_syrk.py $s 3 >> gpurun_out/tma3/syrk_k$k.log 2>&1; done; done
for m in 0 1; do LRGW_TMA_MNCFG=$m timeout 300 python tools/bench_gemm.py path > gpurun_out/tma3/gemm_mn$m.log 2>&1; done
for k in 0 1 2; do LRGW_TMA_KCFG=$k timeout 600 python bench.py --config si64 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tma3/bench_si64_k$k.log 2>&1; done
for k in 0 1 2; do LRGW_TMA_KCFG=$k timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/tma3/bench_si512_k$k.log 2>&1; done
tail -2 gpurun_out/tma3/*.log
