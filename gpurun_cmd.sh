mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py tests/test_gpu_topk.py tests/test_gpu_gw.py -x -q > gpurun_out/fd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fd_tests.log
for f in 1 0; do LRGW_FUSED_DOWNDATE=$f timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fd$f.log 2>&1; done
tail -n 2 gpurun_out/fd_tests.log; for f in 1 0; do echo "fd=$f"; grep -o '"value": [0-9.]*\|"select": [0-9.]*' gpurun_out/bench_fd$f.log | head -3; done
