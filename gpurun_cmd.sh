mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_build.py -x -q -k si512 > gpurun_out/si512_test.log 2>&1; echo "rc=$?" >> gpurun_out/si512_test.log
timeout 300 python tools/fft_probe.py > gpurun_out/fft_probe.log 2>&1
timeout 1200 python bench.py --config si512 --steps 3 --warmup 3 > gpurun_out/bench_si512.log 2>&1; echo "rc=$?" >> gpurun_out/bench_si512.log
tail -3 gpurun_out/si512_test.log; cat gpurun_out/fft_probe.log; tail -c 3000 gpurun_out/bench_si512.log
