"""GPU: the multi-rank build (dist.py) with the device stage backend
(dist_cuda.CudaBackend) on one NCCL rank, against the single-process oracle
— the same checks as the gloo world-2/3 tests (tests/test_dist.py), which
cover the exchange logic on CPU. (This pool gives one GPU per run; ranks that
wait on each other are not stacked on one GPU.)"""
import os
import socket

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

DIMS, CELL = (8, 8, 6), (6.0, 6.0, 4.5)
NV = NC = 8


def _problem():
    rng = np.random.default_rng(11)
    n_r = int(np.prod(DIMS))
    psi = np.linalg.qr(rng.standard_normal((n_r, NV + NC)))[0]
    e = np.concatenate([np.sort(rng.uniform(-0.5, -0.1, NV)), np.sort(rng.uniform(0.05, 0.8, NC))])
    e[NV - 1], e[NV] = -0.1, 0.05
    x = rng.standard_normal((n_r, 3))
    return psi, e, x


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_distributed_build_device_backend_one_rank():
    import torch
    import torch.distributed as dist

    from paper_2403_12340_b200 import dist as D
    from paper_2403_12340_b200.dist_cuda import CudaBackend, _dev

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        psi, e, x = _problem()
        n_mu = R.num_aux(8.0, NV, NC)
        b = D.DistributedBuild(D.Comm(), CudaBackend(n_mu), DIMS, CELL, NV, NC, k_mu=8.0, n_lambda=16, batch=16)
        r0, r1 = b.st.r0, b.st.r1
        pts = b.select(_dev(psi[r0:r1, :NV]), _dev(psi[r0:r1, NV:]))
        theta = b.be.to_host(b.fit(pts))
        t = b.contour(psi[pts, :NV], psi[pts, NV:], e)
        pvp = b.pvp()
        k = b.smw(t, pvp)
        y = b.apply(k, x[r0:r1])
        t, pvp, k = (b.be.to_host(v) for v in (t, pvp, k))
    finally:
        dist.destroy_process_group()
    _check(pts, theta, t, pvp, k, y, psi, e, x)


def _check(pts, theta, t, pvp, k, y, psi, e, x):
    a, bb = psi[:, :NV], psi[:, NV:]
    n_mu = R.num_aux(8.0, NV, NC)
    pts_or = R.select_points(a, bb, n_mu)
    theta_or = R.fit_auxiliary_basis(a, bb, pts_or)
    spec = R.elliptic_params(e, NV, NC, 1e-7)
    t_or = R.coupled_coefficients_fixed(a[pts_or], bb[pts_or], e, spec, 16)
    pvp_or = R.pvp(theta_or, DIMS, CELL)
    k_or = R.assemble_K(t_or, theta_or, DIMS, CELL)
    y_or = R.epsilon_inverse_apply(theta_or, k_or, DIMS, CELL, x)
    rel = lambda u, v: np.linalg.norm(u - v) / np.linalg.norm(v)  # noqa: E731
    assert np.array_equal(pts, pts_or)
    assert rel(theta, theta_or) <= 1e-10
    assert rel(t, t_or) <= 1e-12
    assert rel(pvp, pvp_or) <= 1e-10
    assert rel(k, k_or) <= 1e-10
    assert rel(y, y_or) <= 1e-10


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2403_12340_b200 import dist as D
    from paper_2403_12340_b200.dist_cuda import CudaBackend, _dev

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        psi, e, x = _problem()
        n_mu = R.num_aux(8.0, NV, NC)
        b = D.DistributedBuild(D.Comm(), CudaBackend(n_mu), DIMS, CELL, NV, NC, k_mu=8.0, n_lambda=16, batch=16)
        r0, r1 = b.st.r0, b.st.r1
        pts = b.select(_dev(psi[r0:r1, :NV]), _dev(psi[r0:r1, NV:]))
        theta = b.be.to_host(b.fit(pts))
        t = b.contour(psi[pts, :NV], psi[pts, NV:], e)
        pvp = b.pvp()
        k = b.smw(t, pvp)
        y = b.apply(k, x[r0:r1])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pts=pts, theta=theta, t=b.be.to_host(t),
                 pvp=b.be.to_host(pvp), k=b.be.to_host(k), y=y)
    finally:
        dist.destroy_process_group()


def test_distributed_build_device_backend_two_ranks_gloo(tmp_path):
    """Two ranks over gloo sharing cuda:0: the exchanges are host-side
    collectives (no kernel waits on another rank's kernel); checks the device
    backend's panel / slab / ragged-gather logic at world 2."""
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    psi, e, x = _problem()
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in res:
        assert np.array_equal(r["pts"], res[0]["pts"])
    theta = np.concatenate([r["theta"] for r in res])
    y = np.concatenate([r["y"] for r in res])
    _check(res[0]["pts"], theta, res[1]["t"], res[1]["pvp"], res[1]["k"], y, psi, e, x)
