"""Device stage backend for the multi-rank build (dist.py) on one GPU per rank.

Per-rank arrays (row panels of Phi, L, Theta; the slab spectra) are CUDA
float64 tensors in column-major views; every contraction goes through the
path's kernels: the DMMA GEMM engine (lrgw.dgemm_dev), the candidate scan
(select_topk_dev), the recursive triangular inverse (trtri_lower_dev), the K3
quadrature (contour_partial_dev), the SMW core (smw_core_dev) and the
Coulomb apply. torch.fft (cuFFT) is the FFT leaf; elementwise glue (squares,
row sums, the Hadamard of two GEMM outputs, the spectrum weights) is torch.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import lrgw


def _cm(rows, cols):
    """Zero column-major CUDA float64 matrix (rows x cols)."""
    return torch.zeros(cols, rows, dtype=torch.float64, device="cuda").t()


def _dev(a):
    """numpy (any order) or CUDA tensor -> column-major CUDA float64 tensor."""
    if isinstance(a, torch.Tensor):
        a = a.to("cuda", torch.float64)
        if a.dim() == 1:
            a = a.reshape(-1, 1)
        return a if a.stride(0) == 1 else a.t().contiguous().t()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


class CudaBackend:
    """Stage primitives of dist.DistributedBuild on the local GPU."""

    def __init__(self, n_mu, ctx=None):
        self.n_mu = n_mu
        self.ctx = ctx or lrgw.default_context()

    # ---- arrays -------------------------------------------------------------
    def zeros(self, r, c):
        return _cm(r, c)

    def to_host(self, a):
        return a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)

    def row(self, m, i):
        return m[i].cpu().numpy()

    def rows(self, m, idx):
        """Several local rows at once (one gather + one copy)."""
        ii = torch.as_tensor(np.asarray(idx, dtype=np.int64), device=m.device)
        return m.index_select(0, ii).cpu().numpy()

    # ---- stage 1 --------------------------------------------------------------
    def init_diag(self, a, b):
        return ((a * a).sum(1) * (b * b).sum(1)).contiguous()

    def iota(self, n):
        return torch.arange(n, dtype=torch.int32, device="cuda")

    def local_top(self, d, pos_p, r0, k, s1):
        pos = pos_p.contiguous()
        rows, vals, poss = lrgw.select_topk_dev(d, pos, k, s1, ctx=self.ctx)
        out = []
        for r, v, p in zip(rows.tolist(), vals.tolist(), poss.tolist()):
            out.append((v, p, r0 + r) if r >= 0 else (-math.inf, 2**31 - 1, -1))
        return out

    def cand_greedy(self, top, w_cc, kb, steps, pos, perm):
        """The block's certified greedy on the device (select.cu kernel)."""
        s = len(top) - 1
        x = _cm(s, s)
        b, piv, margins = lrgw.cand_greedy_dev(
            pos.shape[0], steps, kb, [e[0] for e in top], [e[1] for e in top], [e[2] for e in top], _dev(w_cc),
            pos, perm, x, ctx=self.ctx)
        return b, [int(r) for r in piv], x[:b, :b], [float(m) for m in margins]

    def w_panel(self, a, b, amu, bmu, L, lc, k):
        nb = amu.shape[0]
        p1, p2 = _cm(a.shape[0], nb), _cm(a.shape[0], nb)
        lrgw.dgemm_dev("N", "T", 1.0, a, _dev(amu), 0.0, p1, ctx=self.ctx)
        lrgw.dgemm_dev("N", "T", 1.0, b, _dev(bmu), 0.0, p2, ctx=self.ctx)
        w = (p1 * p2).t().contiguous().t()
        if k:
            lrgw.dgemm_dev("N", "T", -1.0, L[:, :k], _dev(lc), 1.0, w, ctx=self.ctx)
        return w

    def l_update(self, w, x, L, k, b):
        lrgw.dgemm_dev("N", "T", 1.0, w, _dev(x), 0.0, L[:, k:k + b], ctx=self.ctx)

    def downdate(self, L, k, b, pos_p, d):
        live = pos_p >= k + b
        blk = L[:, k:k + b]
        d -= torch.where(live, (blk * blk).sum(1), torch.zeros_like(d))

    # ---- stage 2 --------------------------------------------------------------
    def scatter_rows(self, m, local, at, n, cols):
        """n x cols zeros with rows `local` of m placed at rows `at` (the
        owner's contribution to a replicated row set)."""
        out = torch.zeros(n, cols, dtype=torch.float64, device="cuda")
        if len(local):
            li = torch.as_tensor(np.asarray(local, dtype=np.int64), device="cuda")
            ai = torch.as_tensor(np.asarray(at, dtype=np.int64), device="cuda")
            out[ai] = m.index_select(0, li)[:, :cols]
        return out

    def tri_inverse(self, lp):
        x = _dev(lp)
        lrgw.trtri_lower_dev(x, ctx=self.ctx)
        return x

    def theta_panel(self, L, x, colmap):
        out = _cm(L.shape[0], self.n_mu)
        lrgw.theta_from_factor_dev(L, x, colmap, out, ctx=self.ctx)
        return out

    # ---- stage 3 --------------------------------------------------------------
    def contour_partial(self, pv, pc, e, n_lambda, k0, cnt):
        n = pv.shape[0]
        acc = _cm(n, n)
        if cnt > 0:
            lrgw.contour_partial_dev(_dev(pv), _dev(pc), e, n_lambda, k0, cnt, acc, ctx=self.ctx)
        return acc

    def contour_finish(self, acc, e, n_v, n_c):
        spec = lrgw.elliptic_params(e, n_v, n_c, 1e-7)
        pref = 2.0 * math.sqrt(spec.q * spec.big_q) / (math.pi * spec.r)  # contour.hpp:247-248
        t = pref * _dev(acc)
        return _dev(0.5 * (t + t.t()))

    # ---- stages 4-5 -------------------------------------------------------------
    def rfft2_planes(self, theta_p, zl, n2, n1):
        x = theta_p.t().reshape(-1, zl, n2, n1)                   # (n_mu, zl, n2, n1)
        f = torch.fft.rfftn(x, dim=(2, 3))                        # (n_mu, zl, n2, n1h)
        return f.permute(1, 2, 3, 0).contiguous()                 # (zl, n2, n1h, n_mu)

    def y_blocks(self, xh, chunks):
        """The slab spectrum cut into y-chunks, one flat real block per rank."""
        return [torch.view_as_real(xh[:, a:b].contiguous()).reshape(-1) for (a, b) in chunks]

    def z_join(self, recv, planes, tail):
        """Blocks received from every rank -> this rank's y-pencil (n3, ny, n1h, n_mu)."""
        return torch.cat([torch.view_as_complex(r.reshape(-1, 2)).reshape(p, *tail)
                          for r, p in zip(recv, planes)], 0)

    def vcat(self, parts):
        return torch.cat([_dev(p) for p in parts], 0).t().contiguous().t()

    def fft_z(self, pencil):
        g = torch.as_tensor(pencil, device="cuda")
        return torch.fft.fft(g, dim=0)

    def pvp_slab(self, ghat, yr, dims, cell):
        n1, n2, n3 = dims
        n1h = n1 // 2 + 1
        v = lrgw.coulomb_kernel(dims, cell).reshape(n3, n2, n1)[:, yr[0]:yr[1], :n1h]
        herm = np.full(n1h, 2.0)
        herm[0] = 1.0
        if n1 % 2 == 0:
            herm[-1] = 1.0
        w = (v * herm[None, None, :] / (n1 * n2 * n3)).reshape(-1)  # >= 0 (4 pi / |G|^2)
        sw = torch.as_tensor(np.sqrt(w), device="cuda")
        g = ghat.reshape(-1, ghat.shape[-1]) * sw[:, None]          # (K, n_mu) complex
        x = torch.cat([g.real, g.imag], 0)                          # (2K, n_mu) real
        xc = x.t().contiguous().t()
        out = _cm(x.shape[1], x.shape[1])
        lrgw.dgemm_dev("T", "N", 1.0, xc, xc, 0.0, out, ctx=self.ctx)
        return out

    def smw_core(self, t, pvp):
        k = _cm(t.shape[0], t.shape[0])
        p = _dev(pvp)
        lrgw.smw_core_dev(_dev(t), _dev(0.5 * (p + p.t())), k, ctx=self.ctx)
        return k

    def theta_t_x(self, theta, x):
        xd = _dev(x)
        out = _cm(theta.shape[1], xd.shape[1])
        lrgw.dgemm_dev("T", "N", 1.0, theta, xd, 0.0, out, ctx=self.ctx)
        return out

    def theta_w(self, theta, w):
        wd = _dev(w)
        out = _cm(theta.shape[0], wd.shape[1])
        lrgw.dgemm_dev("N", "N", 1.0, theta, wd, 0.0, out, ctx=self.ctx)
        return out

    def apply_coulomb(self, dims, cell, z):
        zd = _dev(z)
        y = _cm(zd.shape[0], zd.shape[1])
        lrgw.coulomb_apply_dev(dims, cell, zd, y, ctx=self.ctx)
        return y
