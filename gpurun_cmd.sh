mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py -x -q -k "not si512" > gpurun_out/h8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h8_tests.log
for w in 1 0; do LRGW_HAD128=$w timeout 600 python tools/trace_build.py si512 2 > gpurun_out/trace512_h$w.log 2>&1; done
timeout 900 python bench.py --config c60 --steps 5 --warmup 3 > gpurun_out/bench_c60.log 2>&1
tail -n 2 gpurun_out/h8_tests.log
for w in 1 0; do echo "== had128_park=$w"; grep -E "^stages|true, 8|128, 64, 32, 32, 4, 2, true" gpurun_out/trace512_h$w.log | cut -c1-150; done
grep -o '"value": [0-9.]*' gpurun_out/bench_c60.log | head -3
