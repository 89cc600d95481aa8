"""CPU: the multi-rank orchestration (paper_2403_12340_b200/dist.py) over gloo
with world sizes 2 and 3 and a numpy stage backend, against the single-process
oracle: bit-exact pivots, Theta / T / Theta^T V Theta / K / eps^-1 x within
1e-10."""
import math
import os
import socket

import numpy as np
import pytest

from oracle import restate as R
from paper_2403_12340_b200 import dist as D


class NumpyBackend:
    """Per-rank stage primitives in numpy (test double of the device backend)."""

    def __init__(self, n_mu):
        self.n_mu = n_mu

    def zeros(self, r, c):
        return np.zeros((r, c))

    def iota(self, n):
        return np.arange(n, dtype=np.int64)

    def init_diag(self, a, b):
        return (a * a).sum(1) * (b * b).sum(1)

    def local_top(self, d, pos_p, r0, k, s1):
        ent = [(float(d[i]), int(pos_p[i]), r0 + i) for i in range(len(d)) if pos_p[i] >= k]
        ent.sort(key=lambda e: (-e[0], e[1]))
        ent = ent[:s1]
        while len(ent) < s1:
            ent.append((-math.inf, 2**31 - 1, -1))
        return ent

    def row(self, m, i):
        return m[i]

    def rows(self, m, idx):
        return m[np.asarray(idx, dtype=np.int64)]

    def rows_cat(self, parts, local, at, n):
        out = np.zeros((n, sum(w for _, w in parts)))
        c0 = 0
        for m, w in parts:
            out[at, c0:c0 + w] = m[local, :w]
            c0 += w
        return out

    def schur_block(self, rc, n1, n2):
        a, b, lc = rc[:, :n1], rc[:, n1:n1 + n2], rc[:, n1 + n2:]
        return (a @ a.T) * (b @ b.T) - lc @ lc.T

    def take_cols(self, m, c0, c1):
        return np.ascontiguousarray(m[:, c0:c1])

    def take_rows(self, m, idx):
        return m[np.asarray(idx, dtype=np.int64)]

    def panel_update(self, a, b, prow, x, L, k, nb, pos_p, d):
        n1, n2 = a.shape[1], b.shape[1]
        w = (a @ prow[:, :n1].T) * (b @ prow[:, n1:n1 + n2].T)
        if k:
            w -= L[:, :k] @ prow[:, n1 + n2:].T
        L[:, k:k + nb] = w @ x.T
        m = pos_p >= k + nb
        d[m] -= (L[m, k:k + nb] ** 2).sum(1)

    def scatter_rows(self, m, local, at, n, cols):
        out = np.zeros((n, cols))
        out[at] = m[local, :cols]
        return out

    def tri_inverse(self, lp):
        import scipy.linalg as sla

        return sla.solve_triangular(np.tril(lp), np.eye(lp.shape[0]), lower=True)

    def theta_panel(self, L, x, colmap):
        xs = np.zeros_like(x)
        xs[:, colmap] = x
        return L[:, :self.n_mu] @ xs

    def contour_partial(self, pv, pc, e, n_lambda, k0, cnt):
        spec = R.elliptic_params(e, pv.shape[1], pc.shape[1], 1e-7)
        nodes, w = R.trapezoid_nodes(spec, n_lambda)
        return R.sum_node_terms(pv, pc, e, spec, nodes[k0:k0 + cnt], w[k0:k0 + cnt])

    def contour_finish(self, acc, e, n_v, n_c):
        spec = R.elliptic_params(e, n_v, n_c, 1e-7)
        return R.symmetrize(R.contour_prefactor(spec) * acc)

    def rfft2_planes(self, theta_p, zl, n2, n1):
        x = theta_p.reshape(zl, n2, n1, -1)
        return np.fft.rfftn(x, axes=(1, 2))

    def y_blocks(self, xh, chunks):
        return [np.ascontiguousarray(xh[:, a:b]).view(np.float64).reshape(-1) for (a, b) in chunks]

    def z_join(self, recv, planes, tail):
        return np.concatenate([r.view(np.complex128).reshape(p, *tail) for r, p in zip(recv, planes)], axis=0)

    def vcat(self, parts):
        return np.concatenate(parts)

    def fft_z(self, pencil):
        return np.fft.fft(pencil, axis=0)

    def pvp_slab(self, ghat, yr, dims, cell):
        n1, n2, n3 = dims
        n1h = n1 // 2 + 1
        v = R.coulomb_kernel(dims, cell).reshape(n3, n2, n1)[:, yr[0]:yr[1], :n1h]
        herm = np.full(n1h, 2.0)
        herm[0] = 1.0
        if n1 % 2 == 0:
            herm[-1] = 1.0
        c = (v * herm[None, None, :] / (n1 * n2 * n3)).reshape(-1)
        g = ghat.reshape(-1, ghat.shape[-1])
        return (g.conj().T @ (c[:, None] * g)).real

    def smw_core(self, t, pvp):
        half = R.symmetrize(0.5 * np.linalg.inv(t))
        return R.symmetrize(np.linalg.inv(half - R.symmetrize(pvp)))

    def theta_t_x(self, theta, x):
        return theta.T @ x

    def matmul(self, a, b):
        return np.asarray(a) @ np.asarray(b)

    def theta_w(self, theta, w):
        return theta @ w

    def apply_coulomb(self, dims, cell, z):
        return R.apply_coulomb(dims, cell, z)

    def to_host(self, a):
        return np.asarray(a)


DIMS, CELL = (8, 8, 6), (6.0, 6.0, 4.5)
NV = NC = 8


def _problem(dims=DIMS):
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


def _worker(rank, world, port, out_dir, dims=DIMS):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        psi, e, x = _problem(dims)
        comm = D.Comm()
        n_mu = R.num_aux(8.0, NV, NC)
        b = D.DistributedBuild(comm, NumpyBackend(n_mu), dims, CELL, NV, NC, k_mu=8.0, n_lambda=16, batch=16)
        r0, r1 = b.st.r0, b.st.r1
        pts = b.select(psi[r0:r1, :NV].copy(), psi[r0:r1, NV:].copy())
        theta_p = b.fit(pts)
        pv, pc = b.point_rows(pts, psi[r0:r1, :NV], psi[r0:r1, NV:])
        assert np.array_equal(pv, psi[pts, :NV]) and np.array_equal(pc, psi[pts, NV:])
        t = b.contour(pv, pc, e)
        pvp = b.pvp()
        k = b.smw(t, pvp)
        y_p = b.apply(k, x[r0:r1])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pts=pts, theta=theta_p, t=t, pvp=pvp, k=k, y=y_p,
                 r0=r0, r1=r1, margins=np.array(b.st.margins))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, DIMS), (3, DIMS), (2, (8, 6, 7))])
def test_distributed_build_matches_oracle(world, dims, tmp_path):
    """(8, 6, 7): ragged z-panels (4 + 3 planes) and y-chunks."""
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), dims), nprocs=world, join=True)
    psi, e, x = _problem(dims)
    a, b = psi[:, :NV], psi[:, NV:]
    n_mu = R.num_aux(8.0, NV, NC)
    pts_or = R.select_points(a, b, n_mu)
    theta_or = R.fit_auxiliary_basis(a, b, pts_or)
    spec = R.elliptic_params(e, NV, NC, 1e-7)
    t_or = R.coupled_coefficients_fixed(a[pts_or], b[pts_or], e, spec, 16)
    pvp_or = R.pvp(theta_or, dims, CELL)
    k_or = R.assemble_K(t_or, theta_or, dims, CELL)
    y_or = R.epsilon_inverse_apply(theta_or, k_or, dims, CELL, x)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    rel = lambda u, v: np.linalg.norm(u - v) / np.linalg.norm(v)  # noqa: E731
    for r in res:
        assert np.array_equal(r["pts"], pts_or), "pivots must be bit-exact across ranks"
        assert rel(r["t"], t_or) <= 1e-12
        assert rel(r["pvp"], pvp_or) <= 1e-10
        assert rel(r["k"], k_or) <= 1e-10
    theta = np.concatenate([r["theta"] for r in res])
    y = np.concatenate([r["y"] for r in res])
    assert rel(theta, theta_or) <= 1e-10
    assert rel(y, y_or) <= 1e-10


def test_partitions_cover_the_grid():
    for world in (1, 2, 3, 4, 8):
        pan = D.z_panels((96, 96, 96), world)
        assert pan[0][0] == 0 and pan[-1][1] == 96 ** 3
        assert all(p[1] == q[0] for p, q in zip(pan, pan[1:]))
        assert all((p[1] - p[0]) % (96 * 96) == 0 for p in pan)
        nr = D.node_ranges(41, world)
        assert nr[0][0] == 0 and nr[-1][1] == 41 and all(p[1] == q[0] for p, q in zip(nr, nr[1:]))


def test_merge_top_is_the_pivot_order():
    ent = [(1.0, 5, 50), (2.0, 9, 90), (2.0, 3, 30), (0.5, 1, 10), (-math.inf, 2**31 - 1, -1)]
    top = D.merge_top(ent, 4)
    assert [e[2] for e in top] == [30, 90, 50, 10]
    assert D.merge_top(ent, 6)[-1][2] == -1
