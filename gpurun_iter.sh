mkdir -p gpurun_out
for r in 1 2; do
QUAD_SWEEP=1 timeout 600 python tools/bench_quad.py si64 c60 si216 si512 > gpurun_out/bench_quad_sweep_$r.log 2>&1
awk '{ if ($0 !~ /rel diff vs cp.async=(0.0e\+00|1.[0-9]e-16) rerun maxabs=0.0e\+00/) print "BAD: "$0 }' gpurun_out/bench_quad_sweep_$r.log
done
sed -E 's/n_mu=[0-9]+ bands=[0-9+]+ nodes=[0-9]+ //' gpurun_out/bench_quad_sweep_2.log | cut -c1-120
timeout 300 python tools/bench_quad.py si64 c60 si216 si512 2>&1 | grep tma | sed -E 's/n_mu=[0-9]+ bands=[0-9+]+ nodes=[0-9]+ //'
timeout 900 python tools/stress_build.py si64 100 2>&1 | tail -1
timeout 900 python tools/stress_build.py si216 10 2>&1 | tail -1
timeout 600 python bench.py --config si64 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_si64_rel.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/bench_si64_rel.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['e2e']['value'], {k:round(v,3) for k,v in d['stages_ms'].items()}); print({k:v.get('frac') for k,v in d['kernels'].items()})
PY
