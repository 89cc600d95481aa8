mkdir -p gpurun_out
for r in 1 2; do
( time timeout 1790 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_reference_wide_$r.log 2>&1 ) 2> gpurun_out/bench_reference_wide_time_$r.log; tail -3 gpurun_out/bench_reference_wide_time_$r.log | head -1; cut -c1-160 gpurun_out/bench_reference_wide_$r.log | tail -1
done
