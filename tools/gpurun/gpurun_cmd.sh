# Round-end style verification on one B200 (used with: gpurun -- 'bash gpurun_cmd.sh')
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -n 3 gpurun_out/gpu_tests.log; tail -n 1 gpurun_out/smoke.log; grep -o '"value": [0-9.]*' gpurun_out/bench.log | head -3
