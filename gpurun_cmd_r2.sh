# Round-2 verification on one B200: GPU tests, smoke, bench lines (Si512 default, Si64, sharded world 1)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_si512.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si512.log
timeout 600 python bench.py --config si64 --steps 20 --warmup 5 > gpurun_out/bench_si64.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_si64.log
timeout 600 python bench.py --config si64 --mode sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_si64_sharded1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_si64_sharded1.log
tail -n 3 gpurun_out/gpu_tests.log; tail -n 2 gpurun_out/smoke.log; grep -ho '"value": [0-9.]*' gpurun_out/bench_*.log | head
