"""Stage times of the multi-rank build (dist.DistributedBuild + the device
backend) on one config: `python tools/dist_time.py --config si64` (world 1)
or under torchrun (one GPU per rank). Prints per-stage wall times (each stage
ends in a device sync + barrier) and the single-GPU lrgw.build time beside."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="si64")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2403_12340_b200 import dist as D
    from paper_2403_12340_b200 import lrgw, synth
    from paper_2403_12340_b200.dist_cuda import CudaBackend

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "RANK" not in os.environ:
        os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[args.config]
    psi = synth.orbitals_device(cfg, seed=1, device=torch.device("cuda", local))
    e = synth.energies(cfg)
    x = synth.probe_host(cfg.n_r)
    comm = D.Comm()
    n_mu = lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)

    def sync():
        torch.cuda.synchronize()
        dist.barrier()

    rows = []
    for rep in range(args.reps):
        b = D.DistributedBuild(comm, CudaBackend(n_mu), cfg.dims, cfg.cell3, cfg.n_v, cfg.n_c, k_mu=cfg.k_mu,
                               n_lambda=cfg.n_lambda, batch=128)
        r0, r1 = b.st.r0, b.st.r1
        t = {}
        sync()
        t0 = time.perf_counter()
        pts = b.select(psi[r0:r1, :cfg.n_v], psi[r0:r1, cfg.n_v:])
        sync(); t["select"] = time.perf_counter()
        b.fit(pts)
        sync(); t["fit"] = time.perf_counter()
        ip = torch.as_tensor(pts.astype(np.int64), device=psi.device)
        pp = psi.index_select(0, ip)
        tc = b.contour(pp[:, :cfg.n_v], pp[:, cfg.n_v:], e)
        sync(); t["contour"] = time.perf_counter()
        pvp = b.pvp()
        sync(); t["pvp"] = time.perf_counter()
        k = b.smw(tc, pvp)
        sync(); t["smw"] = time.perf_counter()
        b.apply(k, x[r0:r1])
        sync(); t["apply"] = time.perf_counter()
        prev, st = t0, {}
        for name, v in t.items():
            st[name] = round((v - prev) * 1e3, 2)
            prev = v
        st["total"] = round((prev - t0) * 1e3, 2)
        rows.append(st)
    ctx = lrgw.Context(local)
    ref = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        torch.cuda.synchronize()
        ref.append((time.perf_counter() - t0) * 1e3)
        ep.close()
    if comm.rank == 0:
        print(json.dumps({"config": cfg.name, "world": comm.world, "dist_ms": rows[-1], "all": rows,
                          "lrgw_build_ms": round(min(ref), 2)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
