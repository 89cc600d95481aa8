mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1500 python tools/make_pivot_fixtures.py c60 si216 --out gpurun_out/golden > gpurun_out/fixtures.log 2>&1
cp gpurun_out/golden/*.npz tests/golden/ 2>/dev/null
LRGW_PARITY_OUT=gpurun_out/parity timeout 2400 python -m pytest tests/test_gpu_configs.py tests/test_gpu_build.py -q -s -rA > gpurun_out/configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/configs.log
tail -5 gpurun_out/fixtures.log; tail -15 gpurun_out/configs.log
