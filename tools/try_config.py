"""One device build of a BASELINE config on cuda:0 with stage times, peak
memory and the size-independent properties (K, T symmetric negative
definite, matrix-free SMW residual). Usage: python tools/try_config.py si512"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from paper_2403_12340_b200 import lrgw, synth  # noqa: E402
from test_gpu_build import L_tensor, _eps_residual  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "si512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.CONFIGS[name]
ctx = lrgw.Context(0)
t0 = time.time()
psi = synth.orbitals_device(cfg)
torch.cuda.synchronize()
print(f"orbitals {psi.shape} in {time.time() - t0:.1f}s; torch reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB",
      flush=True)
e = synth.energies(cfg)
out = {"config": name}
for rep in range(reps):
    t0 = time.time()
    ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                    n_lambda=cfg.n_lambda, ctx=ctx)
    torch.cuda.synchronize()
    wall = time.time() - t0
    st = ctx.stage_ms()
    free, total = torch.cuda.mem_get_info()
    print(f"rep {rep}: wall {wall:.2f}s stages_ms {json.dumps({k: round(v, 2) for k, v in st.items()})} "
          f"free {free / 2**30:.1f}/{total / 2**30:.1f} GiB", flush=True)
    out[f"rep{rep}"] = {"wall_s": wall, "stages_ms": st}
    if rep < reps - 1:
        ep.close()
th_p, k_p, t_p = ep.device_ptrs()
k = L_tensor(k_p, (ep.n_mu, ep.n_mu))
t = L_tensor(t_p, (ep.n_mu, ep.n_mu))
out["k_sym"] = float(torch.linalg.norm(k - k.T) / torch.linalg.norm(k))
out["k_max_eig"] = float(torch.linalg.eigvalsh(k).max())
out["t_max_eig"] = float(torch.linalg.eigvalsh(t).max())
x = torch.randn(8, cfg.n_r, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)).t()
out["smw_residual"] = _eps_residual(lrgw, ctx, ep, cfg, x)
out["n_mu"] = ep.n_mu
out["pts_head"] = [int(p) for p in ep.point_indices[:8]]
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/try_{name}.json", "w") as f:
    json.dump(out, f, indent=1)
