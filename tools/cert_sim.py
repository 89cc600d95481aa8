"""How many pivots per candidate block the selection's certificate admits, as a
function of the candidate-set size s (design probe for the selection blocking;
not part of the product). One exact greedy pivoted Cholesky of the pair Gram
(torch FP64 on the GPU, one column per step) gives the pivot residuals v_t;
then for each s the block loop of select_impl is replayed: at block start k the
candidates are the top-s residuals d_k, tau = the (s+1)-th, and the block
certifies the steps t >= k with v_t > tau (capped).
usage: cert_sim.py [config] [caps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c60"]
    psi = synth.orbitals_device(cfg)
    a, b = psi[:, :cfg.n_v], psi[:, cfg.n_v:]
    n_r = a.shape[0]
    n_mu = lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
    t0 = time.time()
    d0 = (a * a).sum(1) * (b * b).sum(1)
    d = d0.clone()
    L = torch.zeros((n_r, n_mu), dtype=torch.float64, device=a.device)
    v = torch.zeros(n_mu, dtype=torch.float64)
    taken = torch.zeros(n_r, dtype=torch.bool, device=a.device)
    order = []
    for t in range(n_mu):
        dm = torch.where(taken, torch.full_like(d, -float("inf")), d)
        p = int(torch.argmax(dm))
        vp = float(dm[p])
        col = (a @ a[p]) * (b @ b[p])
        if t:
            col -= L[:, :t] @ L[p, :t]
        col /= vp ** 0.5
        L[:, t] = col
        d -= col * col
        taken[p] = True
        v[t] = vp
        order.append(p)
    torch.cuda.synchronize()
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'c60'}: n_r={n_r} n_mu={n_mu} exact greedy {time.time() - t0:.1f} s")
    # residuals at block start k: d0 - sum_{t<k} L[:, t]^2 over untaken rows
    csum = torch.cumsum(L * L, dim=1)
    pos = torch.full((n_r,), n_mu, dtype=torch.long, device=a.device)
    pos[torch.tensor(order, device=a.device)] = torch.arange(n_mu, device=a.device)
    caps = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["96", "128", "256"])]
    for s in (128, 192, 256, 384, 512):
        for cap in caps:
            k, runs = 0, []
            while k < n_mu:
                dk = d0 - (csum[:, k - 1] if k else 0.0)
                dk = torch.where(pos < k, torch.full_like(dk, -float("inf")), dk)
                tau = float(torch.topk(dk, s + 1).values[-1])
                r = 1
                while k + r < n_mu and r < cap and v[k + r] > tau:
                    r += 1
                runs.append(r)
                k += r
            print(f"  s={s:4d} cap={cap:4d}: blocks={len(runs):4d} mean run={sum(runs) / len(runs):6.1f} "
                  f"min={min(runs)} runs[:12]={runs[:12]}")


if __name__ == "__main__":
    main()
