"""GPU: the multi-rank build through the C-ABI (lrgw_build_sharded /
lrgw_eps_apply_sharded over an lrgw_comm) against the single-process
oracle: bit-exact pivots, Theta panels / T / Theta^T V Theta / K / eps^-1 x
within 1e-10.

World 1 runs over a one-rank NCCL communicator (the one-GPU build, bit-equal
to lrgw_build). Worlds 2 and 3 run as separate processes sharing cuda:0 with
the host transport over torch.distributed gloo: every exchange is a host-side
collective between kernel launches, so no kernel waits on another rank's
kernel (this pool lends one GPU per run). Ragged z-panels (7 planes over 3
ranks) and several candidate blocks per selection (batch 16) are covered.
The exchange logic itself is also run on CPU with a numpy backend in
tests/test_dist.py (dist.py, the same scheme in Python)."""
import os
import socket

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

NV = NC = 8
CASES = {"even": ((8, 8, 6), (6.0, 6.0, 4.5)), "ragged": ((8, 6, 7), (6.0, 4.5, 5.25))}


def _problem(dims):
    rng = np.random.default_rng(11)
    n_r = int(np.prod(dims))
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


def _cm(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def _check(pts, theta, t, pvp, k, y, psi, e, x, dims, cell):
    a, bb = psi[:, :NV], psi[:, NV:]
    n_mu = R.num_aux(8.0, NV, NC)
    pts_or = R.select_points(a, bb, n_mu)
    theta_or = R.fit_auxiliary_basis(a, bb, pts_or)
    spec = R.elliptic_params(e, NV, NC, 1e-7)
    t_or = R.coupled_coefficients_fixed(a[pts_or], bb[pts_or], e, spec, 16)
    pvp_or = R.pvp(theta_or, dims, cell)
    k_or = R.assemble_K(t_or, theta_or, dims, cell)
    y_or = R.epsilon_inverse_apply(theta_or, k_or, dims, cell, x)
    rel = lambda u, v: np.linalg.norm(u - v) / np.linalg.norm(v)  # noqa: E731
    assert np.array_equal(pts, pts_or)
    assert rel(theta, theta_or) <= 1e-10
    assert rel(t, t_or) <= 1e-12
    assert rel(pvp, pvp_or) <= 1e-10
    assert rel(k, k_or) <= 1e-10
    assert rel(y, y_or) <= 1e-10


def _run_rank(ctx, comm, dims, cell):
    """One rank's part: its panel in, its Theta panel / eps^-1 x panel out."""
    import torch

    from paper_2403_12340_b200 import lrgw

    psi, e, x = _problem(dims)
    r0, rows = lrgw.z_panel(dims, comm.world, comm.rank)
    ctx.set_select_batch(16)
    ep = lrgw.build_sharded(comm, _cm(psi[r0:r0 + rows, :NV]), _cm(psi[r0:r0 + rows, NV:]), e, dims, cell,
                            k_mu=8.0, n_lambda=16, ctx=ctx)
    inf = ep.info()
    assert inf["n_r"] == int(np.prod(dims)) and inf["min_margin"] > 1e-12
    y_p = _cm(np.zeros((rows, 3)))
    lrgw.eps_apply_sharded(comm, ep, _cm(x[r0:r0 + rows]), y_p)
    theta = _view(inf["theta"], rows, ep.n_mu)
    pvp = _view(inf["pvp"], ep.n_mu, ep.n_mu)
    out = dict(pts=ep.point_indices, theta=theta, t=ep.t, pvp=pvp, k=ep.k, y=y_p.cpu().numpy(),
               blocks=inf["select_blocks"], stage_ms=np.array(list(ctx.stage_ms().values())))
    ep.close()
    torch.cuda.synchronize()
    return out


def _view(ptr, rows, cols):
    import torch

    class _H:
        __cuda_array_interface__ = {"shape": (rows * cols,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_H(), device="cuda").view(cols, rows).t().cpu().numpy()


def test_sharded_world1_nccl_equals_one_gpu_build(ctx):
    """world 1 over a one-rank NCCL communicator is the one-GPU build."""
    from paper_2403_12340_b200 import lrgw

    if not lrgw.L.load().lrgw_nccl_available():
        pytest.fail("libnccl.so.2 not loadable on a GPU box")
    dims, cell = CASES["even"]
    comm = lrgw.Comm.nccl(ctx, 0, 1, lrgw.Comm.nccl_unique_id())
    try:
        res = _run_rank(ctx, comm, dims, cell)
    finally:
        comm.close()
    psi, e, x = _problem(dims)
    ep = lrgw.build(_cm(psi[:, :NV]), _cm(psi[:, NV:]), e, dims, cell, k_mu=8.0, n_lambda=16, ctx=ctx)
    assert np.array_equal(res["pts"], ep.point_indices)
    assert np.array_equal(res["k"], ep.k) and np.array_equal(res["t"], ep.t)
    assert np.array_equal(res["theta"], ep.p_vc)
    _check(res["pts"], res["theta"], res["t"], res["pvp"], res["k"], res["y"], psi, e, x, dims, cell)
    ep.close()


def _worker(rank, world, port, out_dir, case):
    import torch
    import torch.distributed as dist

    from paper_2403_12340_b200 import lrgw

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = lrgw.Context(0)
    comm = lrgw.Comm.from_torch(ctx, transport="host")
    try:
        dims, cell = CASES[case]
        res = _run_rank(ctx, comm, dims, cell)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        comm.close()
        ctx.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "even"), (3, "ragged")])
def test_sharded_build_host_transport(tmp_path, world, case):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world, join=True)
    dims, cell = CASES[case]
    psi, e, x = _problem(dims)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in res[1:]:  # replicated outputs bit-identical across ranks
        for key in ("pts", "t", "pvp", "k"):
            assert np.array_equal(r[key], res[0][key]), key
    assert int(res[0]["blocks"]) > 1
    theta = np.concatenate([r["theta"] for r in res])
    y = np.concatenate([r["y"] for r in res])
    _check(res[0]["pts"], theta, res[0]["t"], res[0]["pvp"], res[0]["k"], y, psi, e, x, dims, cell)
