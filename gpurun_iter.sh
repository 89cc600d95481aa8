mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
( time timeout 1790 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference_default.log 2>&1 ) 2> gpurun_out/bench_reference_time.log; tail -3 gpurun_out/bench_reference_time.log; cut -c1-200 gpurun_out/bench_reference_default.log | tail -1
( time timeout 1790 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default_20_5.log 2>&1 ) 2> gpurun_out/bench_default_time.log; tail -3 gpurun_out/bench_default_time.log; cut -c1-200 gpurun_out/bench_default_20_5.log | tail -1
