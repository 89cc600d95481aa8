mkdir -p gpurun_out/r2c
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r2c/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2c/gpu_tests.log
for b in 16 32 64 128 1024; do LRGW_FFT_BATCH=$b timeout 300 python bench.py --config si64 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2c/fft_si64_b$b.log 2>&1; done
for b in 4 8 16 32 1024; do LRGW_FFT_BATCH=$b timeout 400 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2c/fft_si512_b$b.log 2>&1; done
timeout 2400 python tools/cpu_reference_full.py --out gpurun_out/r2c/cpu_reference_full_si64.json > gpurun_out/r2c/cpu_full.log 2>&1
tail -3 gpurun_out/r2c/gpu_tests.log
