mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_implicit.py tests/test_gpu_build.py -x -q -rf > gpurun_out/implicit_tests.log 2>&1; echo "rc=$?" >> gpurun_out/implicit_tests.log; tail -4 gpurun_out/implicit_tests.log
timeout 600 python bench.py --config si64 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_si64_both.log 2>&1
grep -h '^{' gpurun_out/bench_si64_both.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['theta_implicit']['value'], d['theta_implicit']['stages_ms'])"
