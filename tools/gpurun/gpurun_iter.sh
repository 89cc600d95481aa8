mkdir -p gpurun_out
timeout 900 python tools/stress_build.py si64 150 2>&1 | tail -1
timeout 900 python tools/stress_build.py c60 30 2>&1 | tail -1
timeout 900 python tools/stress_build.py si216 12 2>&1 | tail -1
timeout 1200 python tools/stress_build.py si512 3 2>&1 | tail -1
