timeout 600 python bench.py --config si64 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_si64_pipe.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_si512_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_si512_default.log
grep -h '^{' gpurun_out/bench_si64_pipe.log gpurun_out/bench_si512_default.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:6], 'value', d['value'], 'e2e', d['e2e']['value'], 'serial', d['e2e']['serial_value'], 'implicit', d.get('theta_implicit',{}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d['clocks'])"
tail -2 gpurun_out/bench_si512_default.log | cut -c1-300
