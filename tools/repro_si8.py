import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2403_12340_b200 import lrgw, synth
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "si8"]
psi = synth.orbitals_device(cfg)
e = synth.energies(cfg)
ctx = lrgw.Context(0)
ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda, ctx=ctx)
print("ok", ep.point_indices[:8])
