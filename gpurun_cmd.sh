mkdir -p gpurun_out
timeout 1800 python bench.py --config si512 --steps 3 --warmup 3 > gpurun_out/bench_si512c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_si512c.log
grep -o '"value": [0-9.]*' gpurun_out/bench_si512c.log | head -3
