"""Multi-rank orchestration of the eps^-1 build.

One process per GPU; torch.distributed carries the few exchanges. The large
per-rank arrays (row panels of Phi, L, W, Theta) stay with a *stage backend*
(the device kernels on a GPU rank); this module owns the partitioning and the
deterministic exchange logic:

  stage 1  grid-row panels aligned to z-planes; per candidate block one
           all-gather of the local top-(s+1) lists and owner-contributed rows
           of Phi / L at the candidates (sum of zero-padded contributions:
           exact), the candidates' Schur block W[C, C] and the certified
           greedy replicated on every rank, then the accepted pivots' W
           columns and the L block on the local panel only. Pivots are the
           greedy pivots (reference linalg.hpp:26-111).
  stage 2  Theta panel = L panel L_P^-1 (L_P rows owner-contributed).
  stage 3  quadrature nodes split across ranks, all-reduce of the partial T.
  stage 4-5a  z-slab 3-D FFT: local 2-D transforms, one all-to-all to
           y-pencils, local z transform, local G-slab Theta^T V Theta,
           all-reduce.
  stage 5b SMW core replicated; probe: all-reduce of Theta_p^T x.

`Backend` is the per-rank compute interface; tests inject a numpy backend
(tests/test_dist.py) and run world sizes 2-3 over gloo on CPU. The product
path is the same scheme in C++/CUDA behind the C-ABI (lrgw_build_sharded,
csrc/sharded.cu), which tests/test_gpu_dist.py checks at worlds 1-3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------------------------
# partitioning
# ---------------------------------------------------------------------------

def z_panels(dims, world):
    """Contiguous grid-row ranges [r0, r1) per rank, on z-plane boundaries
    (rows n = i1 + n1 (i2 + n2 i3)); every rank gets >= 1 plane when n3 >= world."""
    n1, n2, n3 = dims
    plane = n1 * n2
    out = []
    for p in range(world):
        z0 = (n3 * p) // world
        z1 = (n3 * (p + 1)) // world
        out.append((z0 * plane, z1 * plane))
    return out


def node_ranges(n_nodes, world):
    """Contiguous quadrature-node ranges [k0, k1) per rank."""
    return [((n_nodes * p) // world, (n_nodes * (p + 1)) // world) for p in range(world)]


def y_chunks(n2, world):
    return [((n2 * p) // world, (n2 * (p + 1)) // world) for p in range(world)]


# ---------------------------------------------------------------------------
# collectives (torch.distributed over numpy payloads; NCCL or gloo)
# ---------------------------------------------------------------------------

class Comm:
    """Thin wrapper: rank/world and the handful of exchanges the build needs.

    Payloads are numpy arrays (small replicated data: candidate lists, rows
    at the pivots) or torch tensors (the per-rank device arrays: partial
    cores, the slab spectra). Tensors stay on the device under NCCL (NVLink)
    and are staged through the host under gloo; every call returns the
    payload's own type (and device)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    @staticmethod
    def _is_tensor(a):
        import torch

        return isinstance(a, torch.Tensor)

    def _t(self, a):
        import torch

        if self._is_tensor(a):
            return a.contiguous().to(self.device)
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def _back(self, t, like):
        if self._is_tensor(like):
            return t.to(like.device)
        return t.cpu().numpy()

    def allreduce_sum(self, a):
        if self.world == 1:
            return a
        t = self._t(a)
        if t is a:
            t = t.clone()
        self.dist.all_reduce(t, group=self.group)
        return self._back(t, a)

    def allgather(self, a, ragged=False):
        """Every rank's `a`; ragged: the leading dimension may differ by rank
        (padded to the largest for the collective, trimmed after)."""
        if self.world == 1:
            return [a]
        t = self._t(a)
        if not ragged:
            out = [torch_empty_like(t) for _ in range(self.world)]
            self.dist.all_gather(out, t, group=self.group)
            return [self._back(o, a) for o in out]
        rows = [int(r[0]) for r in self.allgather(np.array([t.shape[0]], dtype=np.int64))]
        pad = torch_zeros((max(rows),) + tuple(t.shape[1:]), t)
        pad[:t.shape[0]] = t
        out = [torch_empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(out, pad, group=self.group)
        return [self._back(o[:r], a) for o, r in zip(out, rows)]

    def alltoall(self, blocks):
        """blocks[q] (flat) goes to rank q; returns the blocks received from
        each rank. Uses all_to_all when the backend has it, else pairwise
        send/recv."""
        import torch

        send = [self._t(b).reshape(-1) for b in blocks]
        sizes = np.array([int(s.numel()) for s in send], dtype=np.int64)
        shapes = self.allgather(sizes)
        recv = [torch.empty(int(shapes[q][self.rank]), dtype=send[0].dtype, device=self.device)
                for q in range(self.world)]
        try:
            self.dist.all_to_all(recv, send, group=self.group)
        except (RuntimeError, ValueError):
            reqs = []
            for q in range(self.world):
                if q == self.rank:
                    recv[q].copy_(send[q])
                    continue
                reqs.append(self.dist.isend(send[q], q, group=self.group))
                reqs.append(self.dist.irecv(recv[q], q, group=self.group))
            for r in reqs:
                r.wait()
        return [self._back(r, blocks[0]) for r in recv]


def torch_empty_like(t):
    import torch

    return torch.empty_like(t)


def torch_zeros(shape, like):
    import torch

    return torch.zeros(shape, dtype=like.dtype, device=like.device)


# ---------------------------------------------------------------------------
# the certified candidate greedy (replicated, deterministic)
# ---------------------------------------------------------------------------

def better(v1, p1, v2, p2):
    """Reference pivot order: larger residual, then the lower current position
    (strict '>' scan over positions, linalg.hpp:45-48)."""
    return v1 > v2 or (v1 == v2 and p1 < p2)


def merge_top(entries, s1):
    """Global top-s1 of (d, pos, row) entries by the pivot order."""
    ent = [tuple(e) for e in entries if e[2] >= 0]
    ent.sort(key=lambda e: (-e[0], e[1]))
    out = ent[:s1]
    while len(out) < s1:
        out.append((-math.inf, 2**31 - 1, -1))
    return out


def cand_greedy(top, w_cc, kb, steps, pos, perm):
    """Exact greedy steps on the candidate Schur complement (select.cu
    cand_greedy_kernel semantics). top: s+1 entries (d, pos, row); w_cc: s x s.
    Mutates pos/perm (replicated position bookkeeping). Returns
    (b, pivot rows, X = L_sel^-1 (b x b, pivot order), margins); the block's
    L columns are W[:, pivots] X^T."""
    s = len(top) - 1
    tau = top[s][0] if top[s][2] >= 0 else -math.inf
    d = np.array([e[0] for e in top[:s]], dtype=np.float64)
    pc = np.array([e[1] for e in top[:s]], dtype=np.int64)
    rows = np.array([e[2] for e in top[:s]], dtype=np.int64)
    used = rows < 0
    w = np.array(w_cc, dtype=np.float64, copy=True)
    lcols, sel, pivots, margins = [], [], [], []
    tmax = min(s, steps - kb)
    for t in range(tmax):
        best, second, bi = -math.inf, -math.inf, -1
        bp = 2**62
        for i in range(s):
            if used[i]:
                continue
            if better(d[i], pc[i], best, bp):
                second = max(second, best)
                best, bp, bi = d[i], pc[i], i
            else:
                second = max(second, d[i])
        if bi < 0 or not (t == 0 or best > tau):
            break
        k = kb + t
        prow, ppos = int(rows[bi]), int(pc[bi])
        occ = int(perm[k])
        perm[k], perm[ppos] = prow, occ
        pos[prow], pos[occ] = k, ppos
        for i in range(s):
            if rows[i] == occ and i != bi:
                pc[i] = ppos
        pc[bi] = k
        inv = 1.0 / math.sqrt(best) if best > 0 else 0.0
        lpiv = math.sqrt(best) if best > 0 else 0.0
        l = np.where(used, 0.0, w[:, bi] * inv)
        l[bi] = lpiv
        d = np.where(used | (np.arange(s) == bi), d, d - l * l)
        w -= np.outer(l, l)
        used[bi] = True
        lcols.append(l)
        sel.append(bi)
        pivots.append(prow)
        margins.append((best - max(second, tau)) / best if best > 0 else 0.0)
    b = len(sel)
    x = np.zeros((b, b))
    if b:
        lsel = np.array([[lcols[t2][sel[t1]] if t2 <= t1 else 0.0 for t2 in range(b)] for t1 in range(b)])
        for j in range(b):
            for i in range(j, b):
                acc = (1.0 if i == j else 0.0) - float(np.dot(lsel[i, j:i], x[j:i, j]))
                x[i, j] = acc / lsel[i, i] if lsel[i, i] != 0.0 else 0.0
    return b, pivots, x, margins


# ---------------------------------------------------------------------------
# the distributed build
# ---------------------------------------------------------------------------

@dataclass
class RankState:
    r0: int
    r1: int
    d: object = None       # residual diagonal of the panel (backend array)
    L: object = None       # panel x steps factor (backend array)
    theta: object = None   # panel x n_mu
    pivots: list = field(default_factory=list)
    margins: list = field(default_factory=list)


class DistributedBuild:
    """Stages 1-5 across the ranks of `comm` with per-rank `backend`."""

    def __init__(self, comm, backend, dims, cell, n_v, n_c, k_mu=8.0, n_lambda=16, batch=64):
        self.comm, self.be = comm, backend
        self.dims, self.cell = tuple(dims), tuple(cell)
        self.n_r = dims[0] * dims[1] * dims[2]
        self.n_v, self.n_c = n_v, n_c
        from . import lrgw  # num_aux through the C-ABI (llround, isdf.hpp:42-46)

        self.n_mu = min(max(lrgw.num_aux(k_mu, n_v, n_c), 1), self.n_r)
        self.n_lambda = n_lambda
        self.batch = batch
        r0, r1 = z_panels(dims, comm.world)[comm.rank]
        self.st = RankState(r0, r1)

    # ---- owner contributions: rows of a panel array at global row indices --
    def _owned_cat(self, rows, parts):
        """[P_1 | P_2 | ...] at global rows for panel arrays P_i (first w_i
        columns each), owner-contributed and summed in one all-reduce (in the
        backend's memory)."""
        rows = np.asarray(rows, dtype=np.int64)
        at = np.nonzero((rows >= self.st.r0) & (rows < self.st.r1))[0]
        return self.comm.allreduce_sum(self.be.rows_cat(parts, rows[at] - self.st.r0, at, len(rows)))

    def select(self, phi_v_p, phi_c_p):
        """Stage 1 over the local panels (rows [r0, r1) of Phi_v / Phi_c)."""
        be, st = self.be, self.st
        n_r, n1, n2 = self.n_r, self.n_v, self.n_c
        steps = min(self.n_mu, n1 * n2, n_r)
        s = max(1, min(self.batch, n_r))
        # position bookkeeping, replicated (identical updates on every rank)
        pos, perm = be.iota(n_r), be.iota(n_r)
        st.d = be.init_diag(phi_v_p, phi_c_p)
        st.L = be.zeros(st.r1 - st.r0, max(steps, 1))
        k = 0
        while k < steps:
            se = min(s, n_r - k)
            local = be.local_top(st.d, pos[st.r0:st.r1], st.r0, k, se + 1)
            gathered = np.concatenate(self.comm.allgather(np.asarray(local, dtype=np.float64).reshape(-1, 3)))
            top = merge_top([(e[0], int(e[1]), int(e[2])) for e in gathered], se + 1)
            cand = [max(e[2], 0) for e in top[:se]]
            # rows of Phi_v | Phi_c | L[:, :k] at the candidates: one exchange
            rows_c = self._owned_cat(cand, ((phi_v_p, n1), (phi_c_p, n2), (st.L, k)))
            # the candidates' Schur block, replicated (s x s)
            w_cc = be.schur_block(rows_c, n1, n2)
            greedy = getattr(be, "cand_greedy", None) or cand_greedy
            b, piv, x, margins = greedy(top, w_cc, k, steps, pos, perm)
            if b <= 0:
                raise RuntimeError("distributed select: no progress")
            # W columns of the accepted pivots on the local panel, then L block
            # the accepted pivots are candidates: their rows are already here
            at = {top[i][2]: i for i in range(se) if top[i][2] >= 0}
            sel = [at[r] for r in piv]
            be.panel_update(phi_v_p, phi_c_p, be.take_rows(rows_c, sel), x, st.L, k, b, pos[st.r0:st.r1], st.d)
            st.pivots += piv
            st.margins += margins
            k += b
        self.pos, self.perm, self.steps = pos, perm, steps
        return np.sort(be.to_host(perm)[:self.n_mu]).astype(np.int32)

    def point_rows(self, pts, phi_v_p, phi_c_p):
        """Phi_v, Phi_c at the (sorted) interpolation points, replicated on
        every rank (owner-contributed, one all-reduce)."""
        n1, n2 = self.n_v, self.n_c
        rc = self._owned_cat(pts, ((phi_v_p, n1), (phi_c_p, n2)))
        return self.be.take_cols(rc, 0, n1), self.be.take_cols(rc, n1, n1 + n2)

    def fit(self, pts):
        """Stage 2: Theta panel = L panel L_P^-1, columns in sorted-point order.
        L_P (the pivot rows of the factor) is owner-contributed and summed in
        the backend's memory."""
        be, st = self.be, self.st
        if self.steps != self.n_mu:
            raise NotImplementedError("distributed fit needs N_mu <= N_v N_c")
        order = np.asarray(st.pivots, dtype=np.int64)
        mine = np.nonzero((order >= st.r0) & (order < st.r1))[0]
        lp = self.comm.allreduce_sum(be.scatter_rows(st.L, order[mine] - st.r0, mine, self.n_mu, self.n_mu))
        x = be.tri_inverse(lp)
        colmap = np.searchsorted(pts, order)
        st.theta = be.theta_panel(st.L, x, colmap)
        return st.theta

    def contour(self, pv, pc, energies):
        """Stage 3: node-split quadrature + all-reduce (pv, pc replicated)."""
        n_nodes = self.n_lambda + 1
        k0, k1 = node_ranges(n_nodes, self.comm.world)[self.comm.rank]
        part = self.be.contour_partial(pv, pc, energies, self.n_lambda, k0, k1 - k0)
        acc = self.comm.allreduce_sum(part)
        return self.be.contour_finish(acc, energies, self.n_v, self.n_c)

    def pvp(self):
        """Stages 4-5a: slab FFT + G-slab SYRK + all-reduce. The spectra stay
        in the backend's memory: the all-to-all moves them rank to rank."""
        n1, n2, n3 = self.dims
        be, st = self.be, self.st
        z0, z1 = st.r0 // (n1 * n2), st.r1 // (n1 * n2)
        xh = be.rfft2_planes(st.theta, z1 - z0, n2, n1)          # (zl, n2, n1h, n_mu) complex
        chunks = y_chunks(n2, self.comm.world)
        recv = self.comm.alltoall(be.y_blocks(xh, chunks))
        ya, yb = chunks[self.comm.rank]
        planes = [(r1 - r0) // (n1 * n2) for (r0, r1) in z_panels(self.dims, self.comm.world)]
        pencil = be.z_join(recv, planes, (yb - ya, n1 // 2 + 1, self.n_mu))  # (n3, ny, n1h, n_mu)
        ghat = be.fft_z(pencil)
        part = be.pvp_slab(ghat, (ya, yb), self.dims, self.cell)
        return self.comm.allreduce_sum(part)

    def smw(self, t, pvp):
        return self.be.smw_core(t, pvp)

    def apply(self, k, x_p):
        """eps^-1 x on the local panel rows: x_p + (V Theta (K Theta^T x))_p."""
        be, st = self.be, self.st
        u = self.comm.allreduce_sum(be.theta_t_x(st.theta, x_p))
        z_p = be.theta_w(st.theta, be.matmul(k, u))
        z = be.vcat(self.comm.allgather(z_p, ragged=True))
        vz = be.apply_coulomb(self.dims, self.cell, z)
        return be.to_host(x_p) + be.to_host(vz)[st.r0:st.r1]
