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

    def rows_cat(self, parts, local, at, n):
        """n x sum(w) zeros with [P_1 | P_2 | ...][local] placed at rows `at`."""
        width = sum(w for _, w in parts)
        out = torch.zeros(n, width, dtype=torch.float64, device="cuda")
        if len(local):
            li = torch.as_tensor(np.asarray(local, dtype=np.int64), device="cuda")
            ai = torch.as_tensor(np.asarray(at, dtype=np.int64), device="cuda")
            out[ai] = torch.cat([m.index_select(0, li)[:, :w] for m, w in parts if w], 1)
        return out

    def schur_block(self, rc, n1, n2):
        """W[C, C] = (A_C A_C^T) o (B_C B_C^T) - L_C L_C^T on the DMMA engine."""
        rc = _dev(rc)
        s = rc.shape[0]
        p1, p2 = _cm(s, s), _cm(s, s)
        lrgw.dgemm_dev("N", "T", 1.0, rc[:, :n1], rc[:, :n1], 0.0, p1, ctx=self.ctx)
        lrgw.dgemm_dev("N", "T", 1.0, rc[:, n1:n1 + n2], rc[:, n1:n1 + n2], 0.0, p2, ctx=self.ctx)
        w = _dev(p1 * p2)
        if rc.shape[1] > n1 + n2:
            lc = rc[:, n1 + n2:]
            lrgw.dgemm_dev("N", "T", -1.0, lc, lc, 1.0, w, ctx=self.ctx)
        return w

    def take_cols(self, m, c0, c1):
        return _dev(m[:, c0:c1])

    def take_rows(self, m, idx):
        return _dev(m.index_select(0, torch.as_tensor(np.asarray(idx, dtype=np.int64), device=m.device)))

    def panel_update(self, a, b, prow, x, L, k, nb, pos_p, d):
        """W columns of the accepted pivots on the panel, the L block and the
        residual downdate in one call (one host sync)."""
        lrgw.select_panel_update_dev(a, b, L, k, prow, x, pos_p.contiguous(), d, ctx=self.ctx)

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
    # Spectra are kept with N_mu outermost, (n_mu, z, y, x) — each Theta
    # column's slab contiguous, the K-major layout of the single-GPU SYRK.
    def rfft2_planes(self, theta_p, zl, n2, n1):
        x = theta_p.t().reshape(-1, zl, n2, n1)                   # (n_mu, zl, n2, n1), a view
        return torch.fft.rfftn(x, dim=(2, 3))                     # (n_mu, zl, n2, n1h)

    def y_blocks(self, xh, chunks):
        """The slab spectrum cut into y-chunks, one flat real block per rank."""
        return [torch.view_as_real(xh[:, :, a:b].contiguous()).reshape(-1) for (a, b) in chunks]

    def z_join(self, recv, planes, tail):
        """Blocks received from every rank -> this rank's y-pencil (n_mu, n3, ny, n1h)."""
        ny, n1h, n_mu = tail
        return torch.cat([torch.view_as_complex(r.reshape(-1, 2)).reshape(n_mu, p, ny, n1h)
                          for r, p in zip(recv, planes)], 1)

    def vcat(self, parts):
        return torch.cat([_dev(p) for p in parts], 0).t().contiguous().t()

    def fft_z(self, pencil):
        return torch.fft.fft(pencil, dim=1)                       # (n_mu, n3, ny, n1h)

    def pvp_slab(self, ghat, yr, dims, cell):
        n1, n2, n3 = dims
        n1h = n1 // 2 + 1
        v = lrgw.coulomb_kernel(dims, cell).reshape(n3, n2, n1)[:, yr[0]:yr[1], :n1h]
        herm = np.full(n1h, 2.0)
        herm[0] = 1.0
        if n1 % 2 == 0:
            herm[-1] = 1.0
        w = (v * herm[None, None, :] / (n1 * n2 * n3)).reshape(-1)
        w2 = torch.as_tensor(np.repeat(w, 2), device="cuda")     # re / im interleaved
        n_mu = ghat.shape[0]
        x = torch.view_as_real(ghat.contiguous()).reshape(n_mu, -1).t()   # (2K, n_mu) column-major
        out = _cm(n_mu, n_mu)
        lrgw.gram_weighted_dev(x, w2, out, ctx=self.ctx)
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

    def matmul(self, a, b):
        """a b on the DMMA engine (the replicated K u of the probe apply)."""
        ad, bd = _dev(a), _dev(b)
        out = _cm(ad.shape[0], bd.shape[1])
        lrgw.dgemm_dev("N", "N", 1.0, ad, bd, 0.0, out, ctx=self.ctx)
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
