"""Stage times of the device build under environment variants (engine
switches), each variant in its own process so the getenv-latched switches
take effect. Also prints a hash of the selected points so a variant that
moves a pivot is visible.
usage: python tools/env_sweep.py si512 'LRGW_TMA_TALL=0' 'LRGW_TMA_TALL=97' ...
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, hashlib, numpy as np, torch
sys.path.insert(0, %r)
from paper_2403_12340_b200 import lrgw, synth
cfg = synth.CONFIGS[%r]
ctx = lrgw.Context(0)
psi = synth.orbitals_device(cfg)
e = synth.energies(cfg)
rows = []
for rep in range(%d):
    ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                    n_lambda=cfg.n_lambda, ctx=ctx)
    torch.cuda.synchronize()
    st = ctx.stage_ms()
    h = hashlib.sha1(np.ascontiguousarray(ep.point_indices).tobytes()).hexdigest()[:12]
    ep.close()
    rows.append({k: round(v, 2) for k, v in st.items() if v}); rows[-1]["pts"] = h
print("RESULT " + json.dumps(rows[1:] if len(rows) > 1 else rows))
"""


def main():
    cfg = sys.argv[1]
    reps = int(os.environ.get("SWEEP_REPS", "3"))
    for var in sys.argv[2:] or [""]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, reps)], env=env, capture_output=True, text=True,
                           timeout=1800)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(json.dumps({"variant": var, "error": (r.stderr or r.stdout)[-800:]}), flush=True)
            continue
        for row in json.loads(line[0][7:]):
            keep = {k: row[k] for k in ("select", "fit_gemm", "pvp", "contour", "fft", "smw", "cusolver", "total", "pts") if k in row}
            print(json.dumps({"variant": var, **keep}), flush=True)


if __name__ == "__main__":
    main()
