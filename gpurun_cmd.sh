mkdir -p gpurun_out
for w in 0 1; do LRGW_HAD_WIDE=$w timeout 600 python tools/trace_build.py si512 2 > gpurun_out/trace512_w$w.log 2>&1; done
for w in 0 1; do echo "== wide=$w"; grep -E "^stages|true, 16|hadamard" gpurun_out/trace512_w$w.log | cut -c1-150; done
