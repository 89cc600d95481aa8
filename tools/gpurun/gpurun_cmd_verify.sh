# Verification on one B200: GPU tests, smoke, bench lines at every config (default = Si512).
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config si64 --steps 20 --warmup 5 > gpurun_out/bench_si64.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si64.log
timeout 600 python bench.py --config c60 --steps 5 --warmup 3 > gpurun_out/bench_c60.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c60.log
timeout 900 python bench.py --config si216 --steps 5 --warmup 3 > gpurun_out/bench_si216.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si216.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
tail -n 3 gpurun_out/gpu_tests.log; tail -n 2 gpurun_out/smoke.log | cut -c1-200; grep -h '"value"' gpurun_out/bench_*.log | cut -c1-200
