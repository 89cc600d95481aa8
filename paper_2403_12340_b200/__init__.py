"""paper_2403_12340_b200 — B200-native (sm_100a) low-rank dielectric-matrix
inversion of arXiv 2403.12340 behind the reference `lrgw` interface.

    csrc/      hand-written CUDA kernels + the C-ABI (include/lrgw_cuda.h)
    lib/       liblrgw_cuda.so (built in-tree)
    lrgw.py    Python mirror of the reference hot-path API over the C-ABI
    synth.py   seeded synthetic Si-like / C60-like workloads (BASELINE configs)
    dist.py    the multi-rank exchange scheme in Python (numpy stage backend for
               the CPU tests); the product path is lrgw_build_sharded (csrc/sharded.cu)
    driver.py  the reference driver's run / scale commands over the GPU path
"""
from . import lrgw  # noqa: F401  (raises ImportError when the extension is missing)

__all__ = ["lrgw"]
