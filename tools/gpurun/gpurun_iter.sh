for bk in 16 24 32 40 48 64; do LRGW_QUAD_BK=$bk timeout 600 python tools/stress_quad.py si216 60 2>&1 | tail -1; done
for bk in 16 32 64; do LRGW_QUAD_BK=$bk timeout 600 python tools/stress_quad.py si512 6 2>&1 | tail -1; done
timeout 600 python tools/stress_quad.py si64 500 2>&1 | tail -1
timeout 600 python tools/stress_quad.py c60 300 2>&1 | tail -1
