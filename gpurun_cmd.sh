for env in 0 512; do
  LRGW_SYRK_L=$env python tools/bench_syrk.py 1024 115200
  LRGW_SYRK_L=$env python tools/bench_syrk.py 3456 383616 3
  LRGW_SYRK_L=$env python tools/bench_syrk.py 960 256000
done
