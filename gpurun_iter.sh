for sp in 0 1 2 3; do echo -n "kcfg=0 splits=$sp "; LRGW_TMA_KCFG=0 LRGW_TMA_KSPLITS=$sp timeout 300 python tools/bench_syrk.py 8192 903168 3 2>&1 | grep syrk; done
for sp in 0 1 2; do echo -n "kcfg=1 splits=$sp "; LRGW_TMA_KCFG=1 LRGW_TMA_KSPLITS=$sp timeout 300 python tools/bench_syrk.py 8192 903168 3 2>&1 | grep syrk; done
