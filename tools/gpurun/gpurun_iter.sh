mkdir -p gpurun_out
timeout 600 python bench.py --config si64 --mode sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_si64_sharded1.log 2>&1; echo "rc=$?"
timeout 900 python bench.py --config si216 --mode sharded --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_si216_sharded1.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
for f in ['gpurun_out/bench_si64_sharded1.log','gpurun_out/bench_si216_sharded1.log']:
  for l in open(f):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['config'].get('parallelism'), {k:round(v,2) for k,v in d.get('stages_ms',{}).items() if k in ('select','fit_gemm','contour','fft','pvp','smw','total')})
PY
tail -2 gpurun_out/bench_si64_sharded1.log | cut -c1-300
