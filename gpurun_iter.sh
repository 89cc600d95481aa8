timeout 600 ncu --set full --import-source on -k regex:fft_ -c 2 -o gpurun_out/ncu_fft python tools/trace_build.py si64 2 > gpurun_out/ncu_fft.log 2>&1
tail -2 gpurun_out/ncu_fft.log
