timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -rf 2>&1 | tail -2
timeout 600 python bench.py --config si64 --mode sharded --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('sharded x1', d['value'], d['stages_ms'])"
