mkdir -p gpurun_out
timeout 900 python bench.py --config c60 --steps 5 --warmup 3 > gpurun_out/bench_c60.log 2>&1
timeout 1200 python bench.py --config si216 --steps 5 --warmup 3 > gpurun_out/bench_si216.log 2>&1
timeout 1500 python bench.py --config si512 --steps 3 --warmup 3 > gpurun_out/bench_si512b.log 2>&1
for f in bench_c60 bench_si216 bench_si512b; do grep -o '"value": [0-9.]*' gpurun_out/$f.log | head -2; done
